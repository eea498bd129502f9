"""GPU parity: fused fake-quant forward, int8 codes, chains, per-operator
path, synthetic generator — device results vs the CPU oracle, bitwise.

Every device call goes through the C-ABI (libqfb.so) via the Python mirror
of the reference API (paper_2511_12653_b200).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from test_oracle_pinning import ac1_pairs, bits32, same_bits_or_both_nan  # noqa: E402


def to_dev(a, cuda, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(cuda)


def host(t):
    import torch
    return t.detach().to("cpu").to(torch.float32).numpy() if t.dtype == torch.float16 else t.detach().cpu().numpy()


def halfify(orc, a):
    """Round to the binary16 grid (the reference's demote, via the oracle)."""
    return np.array([orc.round_to_half(float(v))[0] for v in np.ravel(a)], dtype=np.float32).reshape(np.shape(a))


# --------------------------------------------------------------- AC1 ---

def test_ac1_random_and_boundaries(qfb, orc, cuda):
    """1e5 random (x, s) pairs + every tie/boundary, bitwise."""
    x, s = ac1_pairs()
    n = x.size
    y = qfb.fake_quantize(to_dev(x.reshape(n, 1), cuda), s.astype(np.float64).tolist())
    _, want = orc.fake_quantize(x, s.astype(np.float64), 1, n, 1)
    same_bits_or_both_nan(host(y).ravel(), want)
    codes = qfb.int8_codes(to_dev(x.reshape(n, 1), cuda), s.astype(np.float64).tolist())
    _, cw = orc.int8_codes(x, s.astype(np.float64), 1, n, 1)
    assert np.array_equal(host(codes).ravel(), cw)


def test_pinned_kats(qfb, cuda):
    # test_quant.cpp:45-68 through the device path
    import torch
    x = torch.tensor([0.0, 200.0, 0.37, 0.005, 0.015, -0.001], device=cuda)
    assert qfb.fake_quantize(x[:1], 0.37)[0].item() == 0.0
    assert qfb.fake_quantize(x[1:2], 1.0)[0].item() == 127.0
    assert qfb.fake_quantize(x[2:3], 0.01)[0].item() == np.float32(np.float32(0.01) * 37)
    assert qfb.fake_quantize(x[3:4], 0.01)[0].item() == 0.0
    assert qfb.fake_quantize(x[4:5], 0.01)[0].item() == np.float32(np.float32(0.01) * 2)
    z = qfb.fake_quantize(x[5:6], 0.5)
    assert bits32(host(z))[0] == 0x80000000   # signed zero
    nanv = qfb.fake_quantize(torch.tensor([float("nan"), float("inf"), -float("inf")], device=cuda), 0.5)
    h = host(nanv)
    assert np.isnan(h[0]) and h[1] == 63.5 and h[2] == -63.5


def test_errors_before_compute(qfb, cuda):
    import torch
    x = torch.ones(4, 3, device=cuda)
    with pytest.raises(qfb.ValueError):
        qfb.fake_quantize(x, 0.0)
    with pytest.raises(qfb.ValueError):
        qfb.fake_quantize(x, -0.5)
    with pytest.raises(qfb.ShapeError):
        qfb.fake_quantize(x, [0.5, 0.5, 0.5])   # per-channel length != dim 0


# ----------------------------------------------------- tensor shapes ---

@pytest.mark.parametrize("shape,axis", [((1, 128, 120, 160), None), ((5, 7, 33), 0),
                                        ((4, 32, 48, 64), 1), ((3, 1, 1), 0), ((1,), None),
                                        ((13, 17), 0), ((2, 6, 5, 3), 1)])
@pytest.mark.parametrize("half", [False, True])
def test_fq_fwd_shapes(qfb, orc, cuda, shape, axis, half):
    import torch
    rng = np.random.default_rng(hash((shape, axis, half)) % 2**32)
    x = rng.normal(0, 1.5, shape).astype(np.float32)
    if half:
        x = x.astype(np.float16).astype(np.float32)   # values on the binary16 grid
    if axis is None:
        s = [0.0315]
        outer, ch, inner = 1, 1, x.size
    else:
        C = shape[axis]
        s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C)).tolist()
        outer = int(np.prod(shape[:axis])) if axis > 0 else 1
        ch, inner = C, int(np.prod(shape[axis + 1:]))
    _, want = orc.fake_quantize(x, s, outer, ch, inner, half=int(half))
    for dt in ([torch.float16, torch.float32] if half else [torch.float32]):
        xd = to_dev(x, cuda, dt)
        y = qfb.fake_quantize(xd, s if axis is not None else s[0],
                              precision=qfb.PREC_HALF if half else qfb.PREC_FULL,
                              channel_axis=axis)
        assert np.array_equal(bits32(host(y).ravel()), bits32(want)), dt


def test_config1_full_size_bitwise(qfb, orc, cuda):
    """BASELINE config 1: per-tensor FP32 on 1x128x120x160 with the
    CounterRng inputs of SURVEY §8d C1, bitwise against the oracle."""
    import torch
    n = 128 * 120 * 160
    x = torch.empty(n, device=cuda)
    qfb.fill_rng(x, seed=1, stream=0, kind=1, lo=1.0)
    xh = orc.fill_rng(n, 1, 0, kind=1, lo=1.0)
    assert np.array_equal(bits32(host(x)), bits32(xh))   # same bytes on both sides
    s = qfb.resolve_scale(qfb.softplus_inv(4.0 / 127.0))
    y = qfb.fake_quantize(x.view(1, 128, 120, 160), s)
    _, want = orc.fake_quantize(xh, [s], 1, 1, n)
    assert np.array_equal(bits32(host(y).ravel()), bits32(want))


def test_unaligned_and_inplace(qfb, orc, cuda):
    import torch
    rng = np.random.default_rng(3)
    x = rng.normal(0, 1, 4099).astype(np.float32)
    base = to_dev(np.concatenate([[0.0], x]).astype(np.float32), cuda)
    xd = base[1:]                     # 4-byte aligned only -> scalar path
    y = qfb.fake_quantize(xd, 0.02)
    _, want = orc.fake_quantize(x, [0.02], 1, 1, x.size)
    assert np.array_equal(bits32(host(y)), bits32(want))
    xi = to_dev(x, cuda)
    qfb.fake_quantize(xi, 0.02, out=xi)   # in place
    assert np.array_equal(bits32(host(xi)), bits32(want))


def test_half_nonfinite_latched(qfb, cuda):
    import torch
    # half bit patterns: 1.0, +NaN, -NaN (payload 0x201), 2.0
    x = torch.tensor([0x3c00, 0x7e01, -0x1ff, 0x4000], dtype=torch.int16).view(torch.float16).to(cuda)
    with pytest.raises(qfb.NonFiniteError):
        qfb.fake_quantize(x, 0.5)
    # the store follows round_to_half: NaN -> +-65504 with the input's sign
    ctx = qfb.default_context(0)
    y = torch.empty_like(x)
    s = torch.tensor([0.5], device=cuda)
    qfb.check(qfb.lib().qfb_fq_fwd(ctx.handle, qfb.F16, x.data_ptr(), y.data_ptr(), 1, 1, 4,
                                   s.data_ptr(), 127, 0))
    with pytest.raises(qfb.NonFiniteError):
        ctx.sync()
    h = y.float().cpu().numpy()
    assert h[1] == 65504.0 and h[2] == -65504.0
    ctx.sync()   # latch cleared


# ------------------------------------------------------------- multi ---

def test_fwd_multi_table(qfb, orc, cuda):
    """Many quant points (incl. 2-output shared points) in one launch."""
    import torch
    rng = np.random.default_rng(8)
    ctx = qfb.default_context(0)
    shapes = [(3, 60, 80), (32, 30, 40), (64, 15, 20), (7, 11, 13), (16, 8, 8), (1, 5, 1)]
    entries, keep, expect = [], [], []
    for i, (C, H, W) in enumerate(shapes):
        x = rng.normal(0, 1, (C, H, W)).astype(np.float32)
        n_out = 2 if i % 2 == 0 else 1
        xd = to_dev(x, cuda)
        d = qfb.CFqDesc()
        d.x = xd.data_ptr()
        d.outer, d.channels, d.inner = 1, C, H * W
        d.n_out, d.q_max, d.flags = n_out, 127, 0
        keep.append(xd)
        for k in range(n_out):
            s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
            sd = torch.tensor([np.float32(v) for v in s], device=cuda)
            yd = torch.empty_like(xd)
            d.y[k] = yd.data_ptr()
            d.scale[k] = sd.data_ptr()
            keep += [sd, yd]
            _, want = orc.fake_quantize(x, s, 1, C, H * W)
            expect.append((yd, want))
        entries.append(d)
    table = (qfb.CFqDesc * len(entries))(*entries)
    before = ctx.launch_count
    qfb.check(qfb.lib().qfb_fq_fwd_multi(ctx.handle, qfb.F32, table, len(entries)))
    assert ctx.launch_count - before == 1
    ctx.sync()
    for yd, want in expect:
        assert np.array_equal(bits32(host(yd).ravel()), bits32(want))


# ------------------------------------------------------------- codes ---

@pytest.mark.parametrize("f16", [False, True])
def test_int8_codes(qfb, orc, cuda, f16):
    import torch
    rng = np.random.default_rng(12)
    x = (rng.normal(0, 3, (8, 64, 24))).astype(np.float32)
    x = x.astype(np.float16).astype(np.float32)
    s = np.exp(rng.uniform(np.log(1e-2), np.log(0.2), 8))
    xd = to_dev(x, cuda, torch.float16 if f16 else torch.float32)
    c = qfb.int8_codes(xd, s.tolist())
    _, want = orc.int8_codes(x, s, 1, 8, 64 * 24)
    assert np.array_equal(host(c).ravel(), want)
    # FQ == s * code
    y = qfb.fake_quantize(to_dev(x, cuda), s.tolist())
    prod = (np.repeat(s.astype(np.float32), 64 * 24) * host(c).ravel().astype(np.float32))
    assert np.array_equal(bits32(host(y).ravel() + 0.0), bits32(prod + 0.0))


# ------------------------------------------------------------- chain ---

@pytest.mark.parametrize("act", [0, 1, 2])
@pytest.mark.parametrize("half", [False, True])
def test_chain(qfb, orc, cuda, act, half):
    import torch
    rng = np.random.default_rng(20 + act)
    C, H, W = 16, 24, 40
    a = rng.normal(0, 2, (C, H, W)).astype(np.float32)
    b = rng.normal(0, 2, (C, H, W)).astype(np.float32)
    if half:
        a, b = a.astype(np.float16).astype(np.float32), b.astype(np.float16).astype(np.float32)
    s0, s1 = 0.03, np.exp(rng.uniform(-6, -2, C)).tolist()
    # per-tensor two outputs
    st, ys, pre = orc.fq_chain(a, b, [[s0], [0.011]], 1, 1, a.size, act=act, half=int(half), preact=True)
    for dt in ([torch.float16, torch.float32] if half else [torch.float32]):
        outs, p = qfb.fq_chain(to_dev(a, cuda, dt), to_dev(b, cuda, dt), scales=(s0, 0.011), act=act,
                               half=half, preact=True)
        assert np.array_equal(bits32(host(p).ravel()), bits32(pre))
        for y, w in zip(outs, ys):
            assert np.array_equal(bits32(host(y).ravel()), bits32(w))
    # per-channel, one output, no b
    st, ys, _ = orc.fq_chain(a, None, [s1], 1, C, H * W, act=act, half=int(half))
    outs, _ = qfb.fq_chain(to_dev(a, cuda), None, scales=(s1,), act=act, half=half, channel_axis=0)
    assert np.array_equal(bits32(host(outs[0]).ravel()), bits32(ys[0]))


@pytest.mark.parametrize("act", [0, 1, 2])
@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_chain_lean_paths(qfb, orc, cuda, act, dtype):
    """The lean chain loop (no demotion, no pre-activation output: the
    config-3 shape) and its exits to the general code: inf/NaN in a or b,
    a + b overflowing float32, |v| beyond the f32 screen, scales outside the
    shortcut's range (1e-30) and large ones (30), GELU at and around +-5,
    signed zeros; two per-channel outputs over rows of 280 / 140 units so
    chunks cross rows."""
    import torch
    rng = np.random.default_rng(50 + act)
    C, H, W = 6, 20, 56
    f16 = dtype == "f16"
    a = rng.normal(0, 3, (C, H, W)).astype(np.float32)
    b = rng.normal(0, 3, (C, H, W)).astype(np.float32)
    a[0, 0, :10] = [5.0, -5.0, np.nextafter(np.float32(5), np.float32(6)), np.nextafter(np.float32(-5), np.float32(-6)),
                    np.nextafter(np.float32(5), np.float32(0)), np.nextafter(np.float32(-5), np.float32(0)),
                    0.0, -0.0, 40.0, -40.0]
    b[0, 0, :10] = 0.0
    a[1, 0, :4] = [np.inf, -np.inf, np.nan, 0.0]
    b[2, 0, :3] = [np.nan, np.inf, -0.0]
    if f16:
        # binary16 storage demotes act(a + b): an inf/NaN operand is the
        # reference's non-finite error (checked below), so finite values here
        a[1, 0, :3] = [65504.0, -65504.0, 0.0]
        b[2, 0, :2] = [-65504.0, 65504.0]
        a[3, 0, :2] = [60000.0, -60000.0]
        b[3, 0, :2] = [60000.0, -60000.0]
        a, b = a.astype(np.float16).astype(np.float32), b.astype(np.float16).astype(np.float32)
    else:
        a[3, 0, :2] = [3e38, -3e38]
        b[3, 0, :2] = [3e38, -3e38]
        a[3, 1, :2] = [1e30, -1e30]
    s0 = np.exp(rng.uniform(-6, -2, C))
    s1 = np.exp(rng.uniform(-6, -2, C))
    s1[4] = 1e-30
    s1[5] = 30.0
    st, want, _ = orc.fq_chain(a, b, [s0, s1], 1, C, H * W, act=act, half=int(f16))
    dt = torch.float16 if f16 else torch.float32
    assert st == 0
    outs, _ = qfb.fq_chain(to_dev(a, cuda, dt), to_dev(b, cuda, dt), scales=(s0.tolist(), s1.tolist()), act=act,
                           half=False, channel_axis=0)
    for y, w in zip(outs, want):
        if f16:  # NaN payloads do not survive torch's half -> float widening
            same_bits_or_both_nan(host(y).ravel(), w)
        else:
            assert np.array_equal(bits32(host(y).ravel()), bits32(w))
    # and with one output, no b (the lean loop's other shape)
    st, want, _ = orc.fq_chain(a, None, [s1], 1, C, H * W, act=act, half=int(f16))
    outs, _ = qfb.fq_chain(to_dev(a, cuda, dt), None, scales=(s1.tolist(),), act=act, half=False, channel_axis=0)
    if f16:
        same_bits_or_both_nan(host(outs[0]).ravel(), want[0])
        # an infinity in a: the oracle and the device both report non-finite
        a[1, 0, 2] = np.inf
        st, _, _ = orc.fq_chain(a, b, [s0], 1, C, H * W, act=act, half=1)
        assert st != 0
        with pytest.raises(qfb.NonFiniteError):
            qfb.fq_chain(to_dev(a, cuda, dt), to_dev(b, cuda, dt), scales=(s0.tolist(),), act=act, half=False,
                         channel_axis=0)
    else:
        assert np.array_equal(bits32(host(outs[0]).ravel()), bits32(want[0]))


def test_gelu_portable_bitwise(qfb, orc, cuda):
    import torch
    rng = np.random.default_rng(4)
    v = np.concatenate([rng.normal(0, 3, 100_000), rng.uniform(-100, 100, 1000),
                        [0.0, -0.0, 1e-30, -1e-30, 88.0, -88.0, 1e30, -1e30]]).astype(np.float32)
    want = np.array([orc.gelu(float(t)) for t in v], dtype=np.float32)
    outs, pre = qfb.fq_chain(to_dev(v, cuda), None, scales=(), act=2, preact=True)
    assert np.array_equal(bits32(host(pre)), bits32(want))
    # the definition is the erf GELU to within 2.1e-6 (degree-12 polynomial Phi)
    ref = 0.5 * v.astype(np.float64) * (1 + np.vectorize(__import__("math").erf)(v / np.sqrt(2)))
    assert np.max(np.abs(want[:101_000] - ref[:101_000])) < 5e-6


# --------------------------------------------------------- per-op ---

@pytest.mark.parametrize("half", [False, True])
def test_perop_equals_fused_device(qfb, orc, cuda, half):
    import torch
    x, s = ac1_pairs(30_000, seed=77)
    if half:
        x = halfify(orc, x)
    n = x.size
    ctx = qfb.default_context(0)
    xd = to_dev(x, cuda)
    sd = torch.tensor(s, device=cuda)
    y1 = torch.empty_like(xd)
    y2 = torch.empty_like(xd)
    tmp = torch.empty(3 * n, device=cuda)
    flags = qfb.FLAG_HALF_GRID if half else 0
    qfb.check(qfb.lib().qfb_fq_fwd(ctx.handle, qfb.F32, xd.data_ptr(), y1.data_ptr(), 1, n, 1,
                                   sd.data_ptr(), 127, flags))
    before = ctx.launch_count
    qfb.check(qfb.lib().qfb_fq_fwd_perop(ctx.handle, qfb.F32, xd.data_ptr(), y2.data_ptr(), 1, n, 1,
                                         sd.data_ptr(), 127, flags, tmp.data_ptr()))
    assert ctx.launch_count - before == 4      # divide, clip, round, multiply
    try:
        ctx.sync()
    except qfb.NonFiniteError:
        assert half
    a, b = host(y1), host(y2)
    same_bits_or_both_nan(a, b)
    _, want = orc.fake_quantize(x, s.astype(np.float64), 1, n, 1, half=int(half))
    same_bits_or_both_nan(a, want)


# ------------------------------------------------------------- rng ---

@pytest.mark.parametrize("kind", [0, 1])
def test_fill_rng_matches_oracle(qfb, orc, cuda, kind):
    import torch
    n = 100_003
    for dt, half in ((torch.float32, 0), (torch.float16, 1)):
        t = torch.empty(n, device=cuda, dtype=dt)
        lo, hi = (-3.0, 5.0) if kind == 0 else (0.5, 0.0)
        qfb.fill_rng(t, seed=9, stream=4, kind=kind, lo=lo, hi=hi, offset=12345)
        want = orc.fill_rng(n, 9, 4, kind=kind, lo=lo, hi=hi, offset=12345, half=half)
        assert np.array_equal(bits32(host(t)), bits32(want))


def test_resolve_scales_device_close(qfb, cuda):
    import torch
    ls = np.concatenate([np.linspace(-40, 40, 997), [-100.0, 100.0, 0.0]])
    d = torch.tensor(ls, device=cuda, dtype=torch.float64)
    s32 = torch.empty(ls.size, device=cuda)
    s64 = torch.empty(ls.size, device=cuda, dtype=torch.float64)
    ch = torch.empty(ls.size, device=cuda, dtype=torch.float64)
    ctx = qfb.default_context(0)
    cfg = qfb.QuantConfig().to_c()
    import ctypes
    qfb.check(qfb.lib().qfb_resolve_scales_dev(ctx.handle, d.data_ptr(), ls.size, ctypes.byref(cfg), 0,
                                               s32.data_ptr(), s64.data_ptr(), ch.data_ptr()))
    ctx.sync()
    hs, hc = qfb.scale_grad_factors(ls.tolist())
    got = s64.cpu().numpy()
    assert np.max(np.abs(got - hs) / np.array(hs)) < 1e-15    # <= a couple of ulp
    assert np.array_equal(s32.cpu().numpy(), np.array(hs, dtype=np.float64).astype(np.float32)) or \
        np.sum(s32.cpu().numpy() != np.array(hs).astype(np.float32)) <= 2
    assert np.max(np.abs(ch.cpu().numpy() - hc)) < 1e-15


@pytest.mark.parametrize("act", [0, 1, 2])
def test_chain_f16_extremes(qfb, orc, cuda, act):
    """binary16 chains through the screened fast path and its exits:
    a + b beyond 65504 (saturating demotion), inf/NaN operands (guarded FQ,
    checked pack, non-finite latch), scales below 2^-80 (guarded FQ), and
    plain FQ of f16 inputs with the same mix."""
    import torch
    rng = np.random.default_rng(31 + act)
    C, H, W = 8, 16, 64
    a = rng.normal(0, 2, (C, H, W)).astype(np.float16).astype(np.float32)
    b = rng.normal(0, 2, (C, H, W)).astype(np.float16).astype(np.float32)
    a[1, :, :8] = 60000.0
    b[1, :, :8] = 60000.0
    a[2, 0, :4] = [65504.0, -65504.0, 0.0, -0.0]
    b[3, 0, :4] = [-0.0, 1.0, -65504.0, 2.0]
    s = np.exp(rng.uniform(-6, -2, C))
    s[4] = 1e-30
    s[5] = 30.0
    st, ys, _ = orc.fq_chain(a, b, [s], 1, C, H * W, act=act, half=1)
    outs, _ = qfb.fq_chain(to_dev(a, cuda, torch.float16), to_dev(b, cuda, torch.float16), scales=(s.tolist(),),
                           act=act, half=True, channel_axis=0)
    assert np.array_equal(bits32(host(outs[0]).ravel()), bits32(ys[0]))
    # plain forward on the same f16 tensor, with infinities (FQ(+-inf) = +-q*s)
    a[2, 0, :2] = [np.inf, -np.inf]
    y = qfb.fake_quantize(to_dev(a, cuda, torch.float16), s.tolist())
    _, want = orc.fake_quantize(a, s, 1, C, H * W, half=1)
    assert np.array_equal(bits32(host(y).ravel()), bits32(want))


@pytest.mark.parametrize("frames", [1, 800])
def test_f32_lean_packed_paths_edge_values(qfb, orc, cuda, frames):
    """The f32 lean loops with packed f32x2 arithmetic (2-stage ring for a
    short launch, 3-stage for a longer one): per-channel rows of ties
    (k + 1/2) * s and their float neighbours, subnormal and tiny x (q0 and
    the residual subnormal), +-0, values at the clip boundary and beyond the
    |x| < s * 2^100 screen, inf/NaN, over scales from 1e-6 to 64 — bitwise
    against the oracle."""
    import torch
    rng = np.random.default_rng(91)
    sp = np.array([1e-6, 1e-4, 0.0315, 0.5, 1.0, 3.0, 64.0, 2.0 ** -100, 2.0 ** 100], dtype=np.float32)
    C = sp.size
    rows = []
    for sv in sp:
        v = []
        for k in list(range(-130, 130)):
            t = np.float32(k + 0.5) * sv
            v += [t, np.nextafter(t, np.float32(np.inf)), np.nextafter(t, np.float32(-np.inf))]
        v += [0.0, -0.0, 1e-45, -1e-45, 1.1754944e-38, -1.1754944e-38, 3e-39, -3e-39, 1e-30, -1e-30,
              np.float32(127) * sv, -np.float32(127) * sv, np.float32(1e30), -np.float32(1e30),
              3.4028235e38, -3.4028235e38, np.inf, -np.inf, np.nan]
        v += list(rng.normal(0, 50, 64) * sv)
        rows.append(np.array(v, dtype=np.float32))
    inner = max(r.size for r in rows)
    inner = (inner + 3) // 4 * 4
    x = np.zeros((C, inner), dtype=np.float32)
    for c, r in enumerate(rows):
        x[c, :r.size] = r
    x = np.tile(x[None], (frames, 1, 1))
    y = qfb.fake_quantize(torch.from_numpy(x).to(cuda), sp.astype(np.float64).tolist(), channel_axis=1)
    _, want = orc.fake_quantize(x.ravel(), sp.astype(np.float64), frames, C, inner)
    assert np.array_equal(bits32(host(y).ravel()), bits32(want))


def test_half_fast_path_all_values(qfb, orc, cuda):
    """Every finite binary16 value through the f16 TMA forward (screened
    fast path: negated-residual quotient without copysign) on 64 per-channel
    scales — from 1e-6 over the 2^-80 fast-path threshold (and one ulp
    below it) to 64 and 65504/127 — bitwise against the oracle."""
    import torch
    bits = np.concatenate([np.arange(0x0000, 0x7c00), np.arange(0x8000, 0xfc00)]).astype(np.uint16)
    xs = bits.view(np.float16).astype(np.float32)
    C = 64
    rng = np.random.default_rng(17)
    sp = [1e-6, 2.0 ** -80, np.nextafter(np.float32(2.0 ** -80), np.float32(0)), 1e-4, 0.0315, 0.5, 1.0, 2.0,
          64.0, 65504.0 / 127, 3e-3, 0.1]
    s = np.array(sp + list(np.exp(rng.uniform(np.log(1e-6), np.log(64.0), C - len(sp)))), dtype=np.float32)
    x = np.tile(xs, (C, 1))
    y = qfb.fake_quantize(torch.from_numpy(x).to(cuda).half(), s.astype(np.float64).tolist())
    _, want = orc.fake_quantize(x.ravel(), s.astype(np.float64), 1, C, xs.size, half=1)
    got = host(y).ravel()
    assert np.array_equal(bits32(got), bits32(want))
