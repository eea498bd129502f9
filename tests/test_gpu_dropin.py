"""The drop-in at the reference's own call sites.

oracle/_ref/dropin_frontend (built by oracle/Makefile from tests/dropin/ and
the reference headers, shipped prebuilt like oracle/_ref/libqfref.so) runs
the reference's forward_train / backward_train (frontend.hpp:103-120,
211-258), run_frontend under every ExecutionPlan knob (exec.hpp:55-65,
435-451) and train_scales (distill.hpp:201-285) twice: stock, and with qfb
substituted at frontend.hpp:112-113 / 221-229 (fake_quantize,
fake_quantize_backward), at run_frontend's run_quant_conv calls and at
train_scales' distill_loss call. Every output — features, descriptors,
each layer's fake-quantized activation and weights, image gradients, all
scale gradients, resolved-scale snapshots, the trained scales and Adam
moments — must be byte-identical (test_frontend.cpp:197-208, 265-290;
test_exec.cpp:110-123).
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_frontend")


@pytest.mark.gpu
def test_reference_call_sites_with_qfb_are_bit_identical():
    assert os.path.exists(BIN), "oracle/_ref/dropin_frontend missing: run `make -C oracle` where /root/reference exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1]
    res = json.loads(line)
    assert r.returncode == 0 and res["ok"], res
    assert res["mismatched"] == 0 and res["blobs"] > 200, res
    # include/qfb.hpp's DeviceView overloads (device buffers, async on the
    # context stream) reproduce the reference's per-channel calls bitwise
    assert res["device_view_blobs"] == 12, res
    calls = res["calls"]
    # every substituted entry point was reached through the reference's code
    assert calls["fake_quantize"] > 0 and calls["fake_quantize_backward"] > 0
    assert calls["run_quant_conv"] > 0 and calls["distill_loss"] > 0
