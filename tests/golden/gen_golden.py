#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Runs the unmodified reference headers compiled from /root/reference
(oracle/_ref/libqfref.so, built by oracle/Makefile) on seeded inputs and
stores inputs + outputs as small fixtures. The fixtures travel with the
repo, so the oracle (tests/test_golden.py, CPU) and the device path
(tests/test_gpu_golden.py) are checked against the reference's own bits
even where the reference tree is absent (the GPU box).

    python tests/golden/gen_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def main():
    ref = oracle.Reference()
    rng = np.random.default_rng(20251112)
    out = {}

    # --- fake_quantize per-channel over [n,1]: AC1-style pairs + boundaries
    n = 20000
    s = np.exp(rng.uniform(np.log(1e-4), np.log(4.0), n)).astype(np.float32)
    x = (rng.uniform(-200, 200, n) * s).astype(np.float32)
    ks = np.array([k + 0.5 for k in range(-128, 128)], dtype=np.float32)
    sb = np.repeat(np.float32(0.0315), ks.size * 3)
    xb = np.concatenate([ks * np.float32(0.0315), np.nextafter(ks * np.float32(0.0315), np.float32(np.inf)),
                         np.nextafter(ks * np.float32(0.0315), np.float32(-np.inf))]).astype(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 3.4028235e38], dtype=np.float32)
    x = np.concatenate([x, xb, special])
    s = np.concatenate([s, sb, np.full(special.size, 0.5, np.float32)])
    st, y = ref.fake_quantize(x, [x.size, 1], s.astype(np.float64), per_channel=True)
    assert st == 0
    st, codes = ref.int8_codes(x, [x.size, 1], s.astype(np.float64), per_channel=True)
    assert st == 0
    out["fq_x"], out["fq_s"], out["fq_y"], out["fq_codes"] = x, s.astype(np.float64), y, codes

    # --- per-tensor half path (EmulatedHalf input)
    xh = rng.normal(0, 2, 4096).astype(np.float16).astype(np.float32)
    st, yh = ref.fake_quantize(xh, [4096], [0.0315], half=1)
    assert st == 0
    out["fqh_x"], out["fqh_y"] = xh, yh

    # --- backward per-tensor and per-channel (shapes [C, HW])
    for tag, shape, pc in (("bwd_pt", (6, 777), False), ("bwd_pc", (12, 1031), True)):
        xx = rng.normal(0, 1.5, shape).astype(np.float32)
        up = rng.normal(0, 1, shape).astype(np.float32)
        ls = rng.uniform(-6, -1, shape[0] if pc else 1)
        if pc:
            ls[1] = -100.0
        st, dx, dls = ref.fq_backward(xx, up, list(shape), ls, per_channel=pc)
        assert st == 0
        out[tag + "_x"], out[tag + "_up"], out[tag + "_ls"] = xx, up, ls
        out[tag + "_dx"], out[tag + "_dls"] = dx, dls

    # --- binary16 rounding
    pats = rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32)
    v = pats.view(np.float32)
    out["half_in"] = v
    out["half_out"] = np.array([ref.round_to_half(float(t))[0] for t in v], dtype=np.float32)

    # --- pairwise sums
    lens = np.array([1, 7, 8, 9, 16, 17, 100, 4095, 4097, 76800], dtype=np.int64)
    arrs = [rng.normal(0, 1, int(k)) * np.exp(rng.uniform(-10, 10, int(k))) for k in lens]
    out["pw_lens"] = lens
    out["pw_data"] = np.concatenate(arrs)
    out["pw_sums"] = np.array([ref.pairwise_sum(a) for a in arrs])

    # --- scale math
    ls = np.concatenate([rng.uniform(-40, 40, 500), [-100.0, 0.0, 100.0, 30.0]])
    out["ls"] = ls
    out["ls_s"] = np.array([ref.resolve_scale(t)[1] for t in ls])
    out["ls_sh"] = np.array([ref.resolve_scale(t, 1)[1] for t in ls])
    out["ls_sig"] = np.array([ref.sigmoid(t) for t in ls])

    # --- counter rng
    idx = np.arange(0, 2000, dtype=np.uint64)
    out["rng_normal"] = np.array([ref.L.ref_rng_normal(1, 0, int(i)) for i in idx])
    out["rng_word"] = np.array([ref.L.ref_rng_word(2024, 3, int(i)) for i in idx], dtype=np.uint64)

    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
