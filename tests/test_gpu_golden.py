"""The DEVICE path against the reference's own outputs (golden vectors made
by the reference compiled from its sources, tests/golden/gen_golden.py)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from test_gpu_fwd import host, to_dev  # noqa: E402

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz"))


def b32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def test_device_fq_equals_reference_bits(qfb, cuda):
    import torch
    x, s = G["fq_x"], G["fq_s"]
    y = qfb.fake_quantize(to_dev(x.reshape(-1, 1), cuda), s.tolist())
    assert np.array_equal(b32(host(y).ravel()), b32(G["fq_y"]))
    c = qfb.int8_codes(to_dev(x.reshape(-1, 1), cuda), s.tolist())
    assert np.array_equal(host(c).ravel(), G["fq_codes"])
    for dt in (torch.float32, torch.float16):
        yh = qfb.fake_quantize(to_dev(G["fqh_x"], cuda, dt), 0.0315, precision=qfb.PREC_HALF)
        assert np.array_equal(b32(host(yh)), b32(G["fqh_y"]))


@pytest.mark.parametrize("tag", ["bwd_pt", "bwd_pc"])
def test_device_bwd_equals_reference_bits(qfb, cuda, tag):
    x, up, ls = G[tag + "_x"], G[tag + "_up"], G[tag + "_ls"]
    log_s = float(ls[0]) if tag == "bwd_pt" else ls.tolist()
    g = qfb.fake_quantize_backward(to_dev(x, cuda), log_s, None, to_dev(up, cuda))
    assert np.array_equal(b32(host(g.d_input).ravel()), b32(G[tag + "_dx"].ravel()))
    assert np.array(g.d_log_scale).tobytes() == G[tag + "_dls"].tobytes()
