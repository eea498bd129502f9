"""Pin the C restatement (oracle/qf_oracle.c) to the reference itself.

Every check compares the oracle bitwise with the UNMODIFIED reference headers
compiled from /root/reference (oracle/_ref/libqfref.so), on the reference's
own known-answer tests (proj/tests/test_quant.cpp, test_tensor.cpp) and on
SPEC.md AC1's stronger random + boundary suite.
CPU only.
"""
import math
import struct

import numpy as np
import pytest

import oracle as O

Q = 127.0


def f32(v):
    return struct.unpack("<f", struct.pack("<f", v))[0]


def bits32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def same_bits_or_both_nan(a, b):
    """Bitwise equality INCLUDING NaN sign and payload: the device emulates
    the host's x86 NaN propagation (qfb_device.cuh quiet_nan / x86_add)."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    assert a.shape == b.shape
    assert np.array_equal(bits32(a), bits32(b))


# --------------------------------------------------------------- scales --

def test_resolve_scale_kats(orc, ref):
    # test_quant.cpp:28-36
    st, s = orc.resolve_scale(0.0)
    assert st == 0 and abs(s - (math.log(2.0) + 1e-8)) <= 1e-12 * s
    assert orc.resolve_scale(-100.0) == (0, 1e-6)
    assert orc.resolve_scale(100.0) == (0, 64.0)
    assert orc.resolve_scale(-100.0, half=1) == (0, 1e-4)
    assert orc.resolve_scale(float("nan"))[0] == 4
    assert ref.resolve_scale(float("nan"))[0] == 4


def test_scale_math_bitwise(orc, ref):
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.uniform(-40, 40, 4000), rng.uniform(-1, 1, 1000),
                         [0.0, -0.0, 29.999, 30.0, 30.0001, -30.0, 700.0, -700.0, 1e-300]])
    for x in xs:
        assert orc.softplus(x) == ref.softplus(x)
        assert orc.sigmoid(x) == ref.sigmoid(x)
        for half in (0, 1):
            assert orc.resolve_scale(x, half) == ref.resolve_scale(x, half)
    for y in np.concatenate([rng.uniform(1e-6, 40, 2000), [1e-300, 30.0, 31.0]]):
        assert orc.softplus_inv(y) == ref.softplus_inv(y)
    assert orc.softplus_inv(0.0)[0] == 2 and ref.softplus_inv(0.0)[0] == 2


def test_config_validation(orc, ref):
    # test_quant.cpp:38-43
    c = O.default_cfg()
    assert orc.L.orc_cfg_validate(c) == 0 and ref.cfg_validate(c) == 0
    c.eps = 1e-3
    assert orc.L.orc_cfg_validate(c) == 2 and ref.cfg_validate(c) == 2
    c = O.default_cfg(bits=1)
    assert orc.L.orc_cfg_validate(c) == 2 and ref.cfg_validate(c) == 2


# ------------------------------------------------------------- scalar FQ --

def test_fq_pinned_kats(orc):
    # test_quant.cpp:45-68
    assert orc.fq_value(0.0, f32(0.37)) == 0.0
    assert orc.fq_value(200.0, 1.0) == 127.0
    assert orc.fq_value(f32(0.37), f32(0.01)) == f32(f32(0.01) * 37.0)
    assert orc.fq_value(f32(0.005), f32(0.01)) == 0.0          # tie -> even
    assert orc.fq_value(f32(0.015), f32(0.01)) == f32(f32(0.01) * 2.0)
    # signed zero survives (SURVEY §8 a2 trap 3)
    assert bits32(orc.fq_value(-0.001, 0.5)) == 0x80000000
    assert math.isnan(orc.fq_value(float("nan"), 0.5))        # NaN-propagating clip
    assert orc.fq_value(float("inf"), 0.5) == 63.5
    assert orc.fq_value(float("-inf"), 0.5) == -63.5


def ac1_pairs(n=100_000, seed=2024):
    """SPEC.md:575 AC1: 1e5 random (x, s) + boundary values x/s in
    {+-0.5, +-1.5, +-q_max +- 0.5}, plus every half-integer code boundary."""
    rng = np.random.default_rng(seed)
    s = np.exp(rng.uniform(np.log(1e-4), np.log(4.0), n)).astype(np.float32)
    x = (rng.uniform(-200.0, 200.0, n) * s).astype(np.float32)
    bs, bx = [], []
    for sv in np.exp(rng.uniform(np.log(1e-4), np.log(4.0), 24)).astype(np.float32):
        ks = [0.5, 1.5, Q - 0.5, Q + 0.5] + [k + 0.5 for k in range(-128, 128)]
        for k in ks:
            for sign in (1.0, -1.0):
                v = np.float32(sign * k) * sv
                for d in (-1, 0, 1):  # the tie itself and its float neighbours
                    bx.append(np.nextafter(v, np.float32(np.inf) * d) if d else v)
                    bs.append(sv)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 1e-45, -1e-45,
                        3.4028235e38, -3.4028235e38, 1.1754944e-38], dtype=np.float32)
    for sv in (np.float32(1e-6), np.float32(0.03125), np.float32(64.0)):
        bx.extend(special)
        bs.extend([sv] * special.size)
    x = np.concatenate([x, np.array(bx, dtype=np.float32)])
    s = np.concatenate([s, np.array(bs, dtype=np.float32)])
    return x, s


def test_ac1_oracle_equals_reference(orc, ref):
    x, s = ac1_pairs()
    n = x.size
    # per-channel over [n, 1]: every element gets its own scale
    st_o, yo = orc.fake_quantize(x, s.astype(np.float64), 1, n, 1)
    st_r, yr = ref.fake_quantize(x, [n, 1], s.astype(np.float64), per_channel=True)
    assert st_o == st_r == 0
    same_bits_or_both_nan(yo, yr)
    _, co = orc.int8_codes(x, s.astype(np.float64), 1, n, 1)
    _, cr = ref.int8_codes(x, [n, 1], s.astype(np.float64), per_channel=True)
    assert np.array_equal(co, cr)
    fin = ~np.isnan(x)
    assert co.min() >= -127 and co.max() <= 127
    # FQ == float(s) * float(code) exactly where finite (test_quant.cpp:135-137)
    assert np.array_equal(bits32(yo[fin] + 0.0), bits32(s[fin] * co[fin].astype(np.float32) + 0.0))


def test_fq_tensor_paths(orc, ref):
    rng = np.random.default_rng(5)
    x = rng.normal(0, 1, (6, 7, 33)).astype(np.float32)
    # per-tensor, full and half
    st1, y1 = orc.fake_quantize(x, [0.031], 1, 1, x.size)
    st2, y2 = ref.fake_quantize(x, list(x.shape), [0.031])
    assert st1 == st2 == 0 and np.array_equal(bits32(y1), bits32(y2))
    xh = np.array([orc.round_to_half(float(v))[0] for v in x.ravel()], dtype=np.float32)
    st1, y1 = orc.fake_quantize(xh, [0.031], 1, 1, x.size, half=1)
    st2, y2 = ref.fake_quantize(xh, list(x.shape), [0.031], half=1)
    assert st1 == st2 == 0 and np.array_equal(bits32(y1), bits32(y2))
    # per-channel axis 0
    sc = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), 6))
    st1, y1 = orc.fake_quantize(x, sc, 1, 6, 7 * 33)
    st2, y2 = ref.fake_quantize(x, list(x.shape), sc, per_channel=True)
    assert st1 == st2 == 0 and np.array_equal(bits32(y1), bits32(y2))
    # errors: non-positive scale -> ValueError (2)
    assert orc.fake_quantize(x, [0.0], 1, 1, x.size)[0] == 2
    assert ref.fake_quantize(x, list(x.shape), [-0.5])[0] == 2
    # half path with NaN: reference throws NonFiniteError (4)
    xn = xh.copy()
    xn[3] = np.nan
    assert orc.fake_quantize(xn, [0.031], 1, 1, x.size, half=1)[0] == 4
    assert ref.fake_quantize(xn, list(x.shape), [0.031], half=1)[0] == 4


def test_perop_equals_fused(orc):
    # exec.hpp:276-342 vs :344-381 (test_exec.cpp:110-123)
    x, s = ac1_pairs(20_000, seed=9)
    _, a = orc.fake_quantize(x, s.astype(np.float64), 1, x.size, 1)
    _, b = orc.fake_quantize_perop(x, s.astype(np.float64), 1, x.size, 1)
    same_bits_or_both_nan(a, b)
    xh = np.array([orc.round_to_half(float(v))[0] for v in x[:5000]], dtype=np.float32)
    _, a = orc.fake_quantize(xh, s[:5000].astype(np.float64), 1, 5000, 1, half=1)
    _, b = orc.fake_quantize_perop(xh, s[:5000].astype(np.float64), 1, 5000, 1, half=1)
    same_bits_or_both_nan(a, b)


# -------------------------------------------------------------- binary16 --

def test_half_kats(orc, ref):
    # test_tensor.cpp:72-96
    assert orc.round_to_half(1.0) == (1.0, 0)
    assert orc.round_to_half(f32(0.1))[0] == 0.0999755859375
    assert orc.round_to_half(70000.0) == (65504.0, 1)
    assert orc.round_to_half(2.9802322e-8)[0] == 0.0          # 2^-25 ties to even
    st, y, ovf = ref.demote_half(np.array([1.0, 0.1, 70000.0, -0.0], dtype=np.float32))
    assert st == 0 and ovf == 1 and y[1] == np.float32(0.0999755859375)


def test_half_bitwise_random_and_special(orc, ref):
    rng = np.random.default_rng(11)
    pats = rng.integers(0, 2**32, 150_000, dtype=np.uint64).astype(np.uint32)
    special = np.array([0x00000000, 0x80000000, 0x7f800000, 0xff800000, 0x7fc00000, 0xffc00000,
                        0x477fe000, 0x477fefff, 0x477ff000, 0x477fffff, 0x33000000, 0x33000001,
                        0x337fffff, 0x38800000, 0x387fffff, 0x00000001, 0x7f7fffff], dtype=np.uint32)
    for p in np.concatenate([pats, special]):
        v = float(np.uint32(p).view(np.float32))
        assert orc.L.orc_f32_to_f16_bits(v) == ref.L.ref_f32_to_f16_bits(v)
        a, sa = orc.round_to_half(v)
        b, sb = ref.round_to_half(v)
        same_bits_or_both_nan([a], [b])
        assert sa == sb
    for h in range(0, 0x10000, 7):
        a = orc.L.orc_f16_bits_to_f32(h)
        b = ref.L.ref_f16_bits_to_f32(h)
        same_bits_or_both_nan([a], [b])


# ----------------------------------------------------------- reductions --

def test_pairwise_sum_bitwise(orc, ref):
    rng = np.random.default_rng(3)
    for n in list(range(0, 70)) + [127, 128, 129, 1000, 4095, 4096, 4097, 65537, 1_000_003]:
        a = rng.normal(0, 1, n) * np.exp(rng.uniform(-20, 20, n))
        assert orc.pairwise_sum(a) == ref.pairwise_sum(a)
    # test_tensor.cpp:105-111: 1e6 x 0.1 vs compensated sum
    a = np.full(1_000_000, np.float32(0.1), dtype=np.float64)
    assert abs(orc.pairwise_sum(a) - math.fsum(a)) / math.fsum(a) < 1e-6


# -------------------------------------------------------------- backward --

@pytest.mark.parametrize("half", [0, 1])
def test_backward_bitwise(orc, ref, half):
    rng = np.random.default_rng(17 + half)
    # per-tensor
    x = rng.normal(0, 2.0, (8, 9, 31)).astype(np.float32)
    up = rng.normal(0, 1.0, x.shape).astype(np.float32)
    if half:
        x = np.array([orc.round_to_half(float(v))[0] for v in x.ravel()], dtype=np.float32).reshape(x.shape)
    ls = [O_sp_inv(0.02)]
    st1, dx1, g1 = orc.fq_backward(x, up, ls, 1, 1, x.size, half=half)
    st2, dx2, g2 = ref.fq_backward(x, up, list(x.shape), ls, per_channel=False, half=half)
    assert st1 == st2 == 0
    assert np.array_equal(bits32(dx1), bits32(dx2))
    assert g1.tobytes() == g2.tobytes()
    # per-channel along axis 0, including a clamped channel (chain 0)
    ls = list(rng.uniform(-6, -1, 8)) + []
    ls[2] = -100.0
    st1, dx1, g1 = orc.fq_backward(x, up, ls, 1, 8, 9 * 31, half=half)
    st2, dx2, g2 = ref.fq_backward(x, up, list(x.shape), ls, per_channel=True, half=half)
    assert st1 == st2 == 0
    assert np.array_equal(bits32(dx1), bits32(dx2))
    assert g1.tobytes() == g2.tobytes()
    assert g1[2] == 0.0


def O_sp_inv(y):
    return math.log(math.expm1(y))


def test_backward_kats(orc):
    # test_quant.cpp:155-186
    ls1 = O_sp_inv(1.0 - 1e-8)
    st, dx, g = orc.fq_backward(np.array([200.0], np.float32), np.array([1.0], np.float32), [ls1], 1, 1, 1)
    assert dx[0] == 0.0
    assert abs(g[0] - 127.0 * orc.sigmoid(ls1)) <= 1e-9 * abs(g[0])
    st, dx, g = orc.fq_backward(np.array([200.0], np.float32), np.array([1.0], np.float32), [-100.0], 1, 1, 1)
    assert g[0] == 0.0
    # masked-out d_input keeps the sign of the upstream: 0.0 * -1 = -0.0
    st, dx, g = orc.fq_backward(np.array([200.0], np.float32), np.array([-1.0], np.float32), [ls1], 1, 1, 1)
    assert bits32(dx)[0] == 0x80000000


def test_backward_outer_accumulation(orc, ref):
    # outer > 1 rows per channel == reference per-frame calls accumulated in
    # frame order (frontend.hpp:222-228)
    rng = np.random.default_rng(23)
    B, C, HW = 3, 4, 50
    x = rng.normal(0, 1, (B, C, HW)).astype(np.float32)
    up = rng.normal(0, 1, (B, C, HW)).astype(np.float32)
    ls = rng.uniform(-5, -2, C)
    _, dx, g = orc.fq_backward(x, up, ls, B, C, HW)
    acc = np.zeros(C)
    for b in range(B):
        _, dxr, gr = ref.fq_backward(x[b], up[b], [C, HW], ls, per_channel=True)
        assert np.array_equal(bits32(dx.reshape(B, C, HW)[b]), bits32(dxr.reshape(C, HW)))
        acc = gr.copy() if b == 0 else acc + gr
    assert g.tobytes() == acc.tobytes()
    # accumulate into an existing gradient
    g0 = rng.normal(0, 1, C)
    _, _, g2 = orc.fq_backward(x, up, ls, B, C, HW, d_log_s=g0, accumulate=1)
    expect = g0.copy()
    for b in range(B):
        _, _, gr = ref.fq_backward(x[b], up[b], [C, HW], ls, per_channel=True)
        expect = expect + gr
    assert g2.tobytes() == expect.tobytes()


# ------------------------------------------------------------- chain/rng --

@pytest.mark.parametrize("half", [0, 1])
def test_chain_equals_reference_composition(orc, ref, half):
    rng = np.random.default_rng(31)
    n = 5000
    a = rng.normal(0, 1, n).astype(np.float32)
    b = rng.normal(0, 1, n).astype(np.float32)
    st, ys, pre = orc.fq_chain(a, b, [[0.03], [0.011]], 1, 1, n, act=1, half=half, preact=True)
    assert st == 0
    st, v = ref.residual_join(a, b, half=half)
    assert np.array_equal(bits32(pre), bits32(v))
    for y, s in zip(ys, (0.03, 0.011)):
        st, r = ref.fake_quantize(v, [n], [s], half=half)
        assert st == 0 and np.array_equal(bits32(y), bits32(r))


def test_rng_bitwise(orc, ref):
    for seed, stream in ((1, 0), (2, 7), (2024, 0), (2**63 + 5, 3)):
        for i in list(range(50)) + [10**9, 2**40 + 3]:
            assert orc.L.orc_rng_word(seed, stream, i) == ref.L.ref_rng_word(seed, stream, i)
            assert orc.L.orc_rng_uniform(seed, stream, i) == ref.L.ref_rng_uniform(seed, stream, i)
            assert orc.L.orc_rng_normal(seed, stream, i) == ref.L.ref_rng_normal(seed, stream, i)
