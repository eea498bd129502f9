"""Oracle pinning for the QAT-step pieces: the C
restatement's distillation loss (oracle/qf_oracle.c orc_distill_pair)
bit-identical to the reference's qf::distill_loss (distill.hpp:126-141,
compiled from its sources) on the reference's own test cases
(test_distill.cpp:24-71) and random shapes; the committed reference-made
vectors (tests/golden/distill_vectors.npz); Adam's restatement against the
update rule of distill.hpp:264-279 (no standalone reference entry point:
pinned by restatement, hand-checked here). CPU only."""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "distill_vectors.npz")


def b32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def same(orc_res, ref_res):
    s1, o1, df1, di1 = orc_res
    s2, o2, df2, di2 = ref_res
    assert s1 == 0 and s2 == 0
    assert o1.tobytes() == o2.tobytes(), (o1, o2)
    assert np.array_equal(b32(df1), b32(df2)) and np.array_equal(b32(di1), b32(di2))


def test_identity_pairs_zero(orc, ref):
    rng = np.random.default_rng(1)
    f = rng.uniform(-1, 1, (4, 3, 3)).astype(np.float32)
    i = rng.uniform(-1, 1, (4, 3, 3)).astype(np.float32)
    r = orc.distill_loss(f, f, i, i, 1.0)
    same(r, ref.distill_loss(f, f, i, i, 1.0))
    assert r[1][0] == 0.0 and r[1][3] == 1.0    # test_distill.cpp:24-32


def test_orthogonal_hand_case(orc, ref):
    fs = np.array([1, 0], np.float32).reshape(2, 1, 1)
    ft = np.array([0, 1], np.float32).reshape(2, 1, 1)
    ii = np.array([0.5, 0.25], np.float32).reshape(2, 1, 1)
    r = orc.distill_loss(fs, ft, ii, ii, 1.0)
    same(r, ref.distill_loss(fs, ft, ii, ii, 1.0))
    assert list(r[1]) == [2.0, 1.0, 0.0, 0.0, 1.0]   # test_distill.cpp:34-46


def test_zero_norm_location_guarded(orc, ref):
    fs = np.array([0, 1, 0, 0.5], np.float32).reshape(2, 2, 1)
    r = orc.distill_loss(fs, fs.copy(), fs, fs.copy(), 1.0)
    same(r, ref.distill_loss(fs, fs.copy(), fs, fs.copy(), 1.0))
    assert r[1][3] == 0.5 and r[2].ravel()[0] == 0.0 and r[2].ravel()[2] == 0.0


@pytest.mark.parametrize("shape_f,shape_i", [((3, 4, 4), (3, 4, 4)), ((1, 1, 1), (2, 1, 3)),
                                             ((8, 17, 9), (16, 5, 5)), ((128, 12, 16), (384, 12, 16)),
                                             ((64, 60, 80), (32, 30, 40))])
@pytest.mark.parametrize("lam", [0.0, 0.7, 1.0])
def test_random_pairs_bitwise(orc, ref, shape_f, shape_i, lam):
    rng = np.random.default_rng(sum(shape_f) + int(10 * lam))
    fs, ft = [rng.normal(0, 1, shape_f).astype(np.float32) for _ in range(2)]
    is_, it = [rng.normal(0, 1, shape_i).astype(np.float32) for _ in range(2)]
    fs.reshape(shape_f[0], -1)[:, 0] = 0.0        # one zero-norm location
    same(orc.distill_loss(fs, ft, is_, it, lam), ref.distill_loss(fs, ft, is_, it, lam))


def test_grad_scale_is_the_trainer_scaling(orc):
    """d * inv in double, rounded to float (distill.hpp:243-246)."""
    rng = np.random.default_rng(9)
    s, t = [rng.normal(0, 1, (5, 7, 3)).astype(np.float32) for _ in range(2)]
    _, _, d1 = orc.distill_pair(s, t, 0.8, 1.0)
    _, _, d15 = orc.distill_pair(s, t, 0.8, 1.0 / 15)
    want = (d1.astype(np.float64) * (1.0 / 15)).astype(np.float32)
    assert np.array_equal(b32(d15), b32(want))


def test_golden_vectors(orc):
    g = np.load(GOLD)
    for k in range(int(g["n_cases"])):
        r = orc.distill_loss(g[f"fs{k}"], g[f"ft{k}"], g[f"is{k}"], g[f"it{k}"], float(g[f"lam{k}"]))
        assert r[1].tobytes() == g[f"out{k}"].tobytes()
        assert np.array_equal(b32(r[2]), b32(g[f"df{k}"])) and np.array_equal(b32(r[3]), b32(g[f"di{k}"]))


def test_adam_restatement(orc):
    rng = np.random.default_rng(4)
    n = 37
    p = rng.normal(-3, 1, n)
    m = rng.normal(0, 1e-3, n)
    v = np.abs(rng.normal(0, 1e-5, n))
    g = rng.normal(0, 1e-2, n)
    b1, b2, lr, eps, t = 0.9, 0.999, 5e-3, 1e-8, 7
    want_p, want_m, want_v = p.copy(), m.copy(), v.copy()
    bc1 = 1.0 - math.pow(b1, t)
    bc2 = 1.0 - math.pow(b2, t)
    for k in range(n):     # distill.hpp:267-278, evaluated in Python doubles
        want_m[k] = b1 * want_m[k] + (1.0 - b1) * g[k]
        want_v[k] = b2 * want_v[k] + (1.0 - b2) * g[k] * g[k]
        want_p[k] -= lr * (want_m[k] / bc1) / (math.sqrt(want_v[k] / bc2) + eps)
    assert orc.adam(p, m, v, g, b1, b2, lr, eps, t) == 0
    assert p.tobytes() == want_p.tobytes() and m.tobytes() == want_m.tobytes() and v.tobytes() == want_v.tobytes()
    g2 = g.copy()
    g2[5] = np.nan
    p0 = p.copy()
    assert orc.adam(p, m, v, g2, b1, b2, lr, eps, t + 1) == 1 and p.tobytes() == p0.tobytes()
