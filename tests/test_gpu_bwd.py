"""GPU parity: scale-only STE/LSQ backward vs the CPU oracle.

Bar: d_input bitwise; d_log_s BITWISE as well (the device reproduces the
reference's pairwise tree exactly). The north-star tolerance (rel 1e-5 FP32,
1e-2 FP16) is also asserted explicitly as the contractual floor.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from test_gpu_fwd import bits32, host, to_dev  # noqa: E402

TOL_F32 = 1e-5   # north_star: scale gradients within rel 1e-5 (FP32)
TOL_F16 = 1e-2   # ... and 1e-2 (FP16)


def sp_inv(y):
    return math.log(math.expm1(y))


def check_grads(got, want, tol):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    denom = np.maximum(np.abs(want), 1e-300)
    assert np.all(np.abs(got - want) <= tol * denom + 1e-300), (got, want)
    assert got.tobytes() == want.tobytes()   # bit-exact (stronger than tol)


LENGTHS = [1, 2, 7, 8, 9, 15, 16, 17, 31, 33, 100, 255, 256, 257, 1000, 2816, 3328, 3584, 4095,
           4096, 4097, 4099, 8193, 12288, 65537, 76800]   # leaf groups of every size 1..16


@pytest.mark.parametrize("n", LENGTHS)
def test_per_tensor_ragged_lengths(qfb, orc, cuda, n):
    rng = np.random.default_rng(n)
    s = 0.02
    x = (rng.normal(0, 1, n) * 100 * s).astype(np.float32)   # plenty saturated
    up = rng.normal(0, 1, n).astype(np.float32)
    ls = sp_inv(s)
    g = qfb.fake_quantize_backward(to_dev(x, cuda), ls, None, to_dev(up, cuda))
    _, dx, dls = orc.fq_backward(x, up, [ls], 1, 1, n)
    assert np.array_equal(bits32(host(g.d_input)), bits32(dx))
    check_grads(g.d_log_scale, dls, TOL_F32)


@pytest.mark.parametrize("shape", [(32, 3, 7, 7), (64, 32, 3, 3), (64, 32, 1, 1), (384, 64, 1, 1),
                                   (128, 120, 160), (5, 1)])
def test_per_channel_axis0(qfb, orc, cuda, shape):
    """Weights [C_out, per] and activation maps [C, H*W] (quant.hpp:261)."""
    rng = np.random.default_rng(sum(shape))
    C = shape[0]
    per = int(np.prod(shape[1:]))
    ls = rng.uniform(-6, -1, C)
    ls[0] = -100.0      # clamp-gated channel: chain 0
    x = rng.normal(0, 0.5, shape).astype(np.float32)
    up = rng.normal(0, 1, shape).astype(np.float32)
    g = qfb.fake_quantize_backward(to_dev(x, cuda), ls.tolist(), None, to_dev(up, cuda))
    _, dx, dls = orc.fq_backward(x, up, ls, 1, C, per)
    assert np.array_equal(bits32(host(g.d_input).ravel()), bits32(dx))
    check_grads(g.d_log_scale, dls, TOL_F32)
    assert g.d_log_scale[0] == 0.0


def test_frames_outer_accumulation(qfb, orc, cuda):
    """[B, C, HW] per-channel over frames: rows accumulate in frame order."""
    rng = np.random.default_rng(5)
    B, C, H, W = 4, 32, 30, 40
    x = rng.normal(0, 1, (B, C, H, W)).astype(np.float32)
    up = rng.normal(0, 1, (B, C, H, W)).astype(np.float32)
    ls = rng.uniform(-6, -2, C)
    g = qfb.fake_quantize_backward(to_dev(x, cuda), ls.tolist(), None, to_dev(up, cuda), channel_axis=1)
    _, dx, dls = orc.fq_backward(x, up, ls, B, C, H * W)
    assert np.array_equal(bits32(host(g.d_input).ravel()), bits32(dx))
    check_grads(g.d_log_scale, dls, TOL_F32)


def test_accumulate_and_null_dx(qfb, orc, cuda):
    import torch
    rng = np.random.default_rng(9)
    B, C, HW = 3, 8, 5000
    x = rng.normal(0, 1, (B, C, HW)).astype(np.float32)
    up = rng.normal(0, 1, (B, C, HW)).astype(np.float32)
    ls = rng.uniform(-5, -2, C)
    g0 = rng.normal(0, 1, C)
    s64, chain = qfb.scale_grad_factors(ls.tolist())
    fac = torch.tensor(s64 + chain, dtype=torch.float64, device=cuda)
    dls = torch.tensor(g0, dtype=torch.float64, device=cuda)
    ctx = qfb.default_context(0)
    xd, ud = to_dev(x, cuda), to_dev(up, cuda)
    for _ in range(2):   # twice: the self-resetting tickets must be clean
        qfb.check(qfb.lib().qfb_fq_bwd(ctx.handle, qfb.F32, xd.data_ptr(), ud.data_ptr(), None, B, C, HW,
                                       fac.data_ptr(), fac.data_ptr() + 8 * C, 127, dls.data_ptr(), 1))
    ctx.sync()
    _, _, want = orc.fq_backward(x, up, ls, B, C, HW, d_log_s=g0, accumulate=1, want_dx=False)
    _, _, want = orc.fq_backward(x, up, ls, B, C, HW, d_log_s=want, accumulate=1, want_dx=False)
    check_grads(dls.cpu().numpy(), want, TOL_F32)


def test_half_io(qfb, orc, cuda):
    """FP16 storage: x and upstream on the binary16 grid, s_min_half bound."""
    import torch
    rng = np.random.default_rng(13)
    C, H, W = 64, 60, 80
    x = rng.normal(0, 1, (C, H, W)).astype(np.float16).astype(np.float32)
    up = rng.normal(0, 1, (C, H, W)).astype(np.float16).astype(np.float32)
    ls = rng.uniform(-7, -2, C)
    ls[3] = -100.0
    g = qfb.fake_quantize_backward(to_dev(x, cuda, torch.float16), ls.tolist(), None,
                                   to_dev(up, cuda, torch.float16), precision=qfb.PREC_HALF)
    _, dx, dls = orc.fq_backward(x, up, ls, 1, C, H * W, half=1)
    assert np.array_equal(bits32(host(g.d_input).ravel()), bits32(dx))
    check_grads(g.d_log_scale, dls, TOL_F16)


def test_kats(qfb, cuda):
    # test_quant.cpp:155-186 through the device
    import torch
    ls1 = sp_inv(1.0 - 1e-8)
    g = qfb.fake_quantize_backward(torch.tensor([200.0], device=cuda), ls1, None,
                                   torch.tensor([1.0], device=cuda))
    assert g.d_input.item() == 0.0
    assert abs(g.d_log_scale[0] - 127.0 * qfb.sigmoid(ls1)) <= 1e-9 * abs(g.d_log_scale[0])
    g = qfb.fake_quantize_backward(torch.tensor([200.0], device=cuda), -100.0, None,
                                   torch.tensor([1.0], device=cuda))
    assert g.d_log_scale[0] == 0.0
    g = qfb.fake_quantize_backward(torch.tensor([200.0], device=cuda), ls1, None,
                                   torch.tensor([-1.0], device=cuda))
    assert bits32(host(g.d_input))[0] == 0x80000000   # 0.0 * -1 keeps the sign
    # in range: pass-through
    x = torch.linspace(-0.4, 0.4, 64, device=cuda)
    g = qfb.fake_quantize_backward(x, sp_inv(0.01), None, torch.ones(64, device=cuda))
    assert torch.all(g.d_input == 1.0)


def test_scale_grad_matches_finite_difference(qfb, cuda):
    """SPEC AC6 / test_quant.cpp:188-236: analytic LSQ grad vs central FD of
    the STE surrogate, rel 1e-4, 40 trials x 96 elements."""
    import torch
    rng = np.random.default_rng(404)
    cfg = qfb.QuantConfig()
    for trial in range(40):
        log_s = rng.uniform(-5.0, 0.5)
        s0 = qfb.resolve_scale(log_s)
        k = np.floor(rng.uniform(0, 140, 96))
        frac = rng.uniform(0.05, 0.45, 96)
        flip = rng.integers(0, 4, 96)
        frac = np.where(flip & 1, frac + 0.54, frac)
        z = k + frac
        z = np.where(np.abs(z - 127) < 0.2, z + 0.5, z)
        z = np.where(flip & 2, -z, z)
        x = (z * s0).astype(np.float32)
        up = rng.uniform(-1, 1, 96).astype(np.float32)
        g = qfb.fake_quantize_backward(torch.tensor(x, device=cuda), log_s, cfg, torch.tensor(up, device=cuda))

        def surrogate(ls):
            s = qfb.resolve_scale(ls)
            xs = x.astype(np.float64)
            z0 = xs / s0
            y = np.where(np.abs(z0) <= 127, xs + (np.rint(z0) - z0) * s, np.sign(z0) * 127 * s)
            return float(np.sum(up.astype(np.float64) * y))
        fd = (surrogate(log_s + 1e-5) - surrogate(log_s - 1e-5)) / 2e-5
        assert abs(g.d_log_scale[0] - fd) <= 1e-4 * abs(fd) + 1e-10


def test_bwd_multi_table_and_determinism(qfb, orc, cuda):
    """All activation quant points of a frame in one launch; run twice,
    identical bits (fixed schedule, any grid)."""
    import torch
    rng = np.random.default_rng(21)
    ctx = qfb.default_context(0)
    shapes = [(3, 120, 160), (32, 60, 80), (32, 60, 80), (64, 30, 40), (64, 30, 40), (7, 9, 11)]
    entries, keep, expect = [], [], []
    for C, H, W in shapes:
        x = rng.normal(0, 1, (C, H, W)).astype(np.float32)
        up = rng.normal(0, 1, (C, H, W)).astype(np.float32)
        ls = rng.uniform(-6, -2, C)
        s64, chain = qfb.scale_grad_factors(ls.tolist())
        fac = torch.tensor(s64 + chain, dtype=torch.float64, device=cuda)
        xd, ud = to_dev(x, cuda), to_dev(up, cuda)
        dx = torch.empty_like(xd)
        dls = torch.zeros(C, dtype=torch.float64, device=cuda)
        d = qfb.CBwdDesc()
        d.x, d.up, d.dx = xd.data_ptr(), ud.data_ptr(), dx.data_ptr()
        d.scale64, d.chain, d.d_log_s = fac.data_ptr(), fac.data_ptr() + 8 * C, dls.data_ptr()
        d.outer, d.channels, d.inner, d.q_max, d.accumulate = 1, C, H * W, 127, 0
        entries.append(d)
        keep += [fac, xd, ud]
        _, wdx, wdls = orc.fq_backward(x, up, ls, 1, C, H * W)
        expect.append((dx, dls, wdx, wdls))
    table = (qfb.CBwdDesc * len(entries))(*entries)
    results = []
    for rep in range(2):
        before = ctx.launch_count
        qfb.check(qfb.lib().qfb_fq_bwd_multi(ctx.handle, qfb.F32, table, len(entries)))
        assert ctx.launch_count - before == 2    # main pass + finisher
        ctx.sync()
        results.append([e[1].cpu().numpy().tobytes() for e in expect])
        for dx, dls, wdx, wdls in expect:
            assert np.array_equal(bits32(host(dx).ravel()), bits32(wdx))
            check_grads(dls.cpu().numpy(), wdls, TOL_F32)
    assert results[0] == results[1]


def test_special_values_bitwise(qfb, orc, cuda):
    """inf / NaN / +-0 / subnormal / huge x and +-inf / NaN upstream through
    the fast two-correction quotient, its IEEE exits and the x86 NaN rules of d_input."""
    rng = np.random.default_rng(77)
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.17e-38, 3.4e38, -3.4e38,
                   0.5, -0.5, 1.5, 127.0, 127.5, -127.5, 126.5, 1e-8], dtype=np.float32)
    for s in (1e-6, 0.0315, 1.0, 2.0, 64.0, 0.5):
        x = np.concatenate([sp * np.float32(s), sp, rng.normal(0, 50 * s, 5000).astype(np.float32)])
        up = rng.normal(0, 1, x.size).astype(np.float32)
        up[::97] = np.inf
        up[1::97] = -np.inf
        up[2::97] = np.nan
        up[3::97] = -0.0
        ls = float(np.log(np.expm1(s))) if s < 30 else s
        g = qfb.fake_quantize_backward(to_dev(x, cuda), ls, None, to_dev(up, cuda))
        _, dx, dls = orc.fq_backward(x, up, [ls], 1, 1, x.size)
        assert np.array_equal(bits32(host(g.d_input)), bits32(dx)), s
        assert np.isnan(g.d_log_scale[0]) and np.isnan(dls[0])
        # finite upstream: gradient bitwise too
        up2 = np.nan_to_num(up, nan=0.5, posinf=2.0, neginf=-2.0)
        g = qfb.fake_quantize_backward(to_dev(x, cuda), ls, None, to_dev(up2, cuda))
        _, dx, dls = orc.fq_backward(x, up2, [ls], 1, 1, x.size)
        assert np.array_equal(bits32(host(g.d_input)), bits32(dx)), s
        check_grads(g.d_log_scale, dls, TOL_F32)


def test_special_values_half_storage(qfb, orc, cuda):
    """The same specials on binary16 storage: +-inf / NaN x and upstream in
    rows long enough for the unrolled leaf groups (9/10 elements), per
    channel; d_input equal (NaN where the reference has NaN), finite-upstream
    scale gradients bitwise."""
    import torch
    rng = np.random.default_rng(78)
    C, n = 4, 6000
    x = rng.normal(0, 2, (C, n)).astype(np.float16).astype(np.float32)
    x[:, ::101] = np.inf
    x[:, 1::101] = -np.inf
    x[:, 2::101] = np.nan
    x[:, 3::101] = -0.0
    up = rng.normal(0, 1, (C, n)).astype(np.float16).astype(np.float32)
    ls = rng.uniform(-4, -1, C)
    for nonfinite_up in (True, False):
        u = up.copy()
        if nonfinite_up:
            u[:, 5::89] = np.inf
            u[:, 6::89] = -np.inf
            u[:, 7::89] = np.nan
        xd = torch.from_numpy(x).to(cuda).half()
        ud = torch.from_numpy(u).to(cuda).half()
        g = qfb.fake_quantize_backward(xd, ls.tolist(), None, ud)
        _, dx, dls = orc.fq_backward(x, u, ls, 1, C, n)
        got = host(g.d_input.float()).ravel()
        nan_w = np.isnan(dx)
        assert np.array_equal(np.isnan(got), nan_w)
        assert np.array_equal(bits32(got[~nan_w]), bits32(dx[~nan_w]))
        if nonfinite_up:
            assert np.array_equal(np.isnan(np.asarray(g.d_log_scale)), np.isnan(dls))
        else:
            check_grads(g.d_log_scale, dls, TOL_F16)


@pytest.mark.parametrize("half", [0, 1])
def test_relu_activations_bitwise(qfb, orc, cuda, half):
    """Post-ReLU conv inputs (about half the elements +-0, the zeros taking
    the exact fast path) at a DPVO layer-2 shape, per channel, f32 and f16
    storage: d_input and d_log_s bitwise."""
    import torch
    rng = np.random.default_rng(11 + half)
    C, H, W = 64, 120, 160
    x = np.maximum(rng.normal(0, 1, (C, H, W)), 0).astype(np.float32)
    x[:, ::7, :] = -0.0
    up = rng.normal(0, 1, (C, H, W)).astype(np.float32)
    if half:
        x = x.astype(np.float16).astype(np.float32)
        up = up.astype(np.float16).astype(np.float32)
    ls = rng.uniform(-6, -2, C)
    dt = torch.float16 if half else torch.float32
    xd = torch.from_numpy(x).to(cuda).to(dt)
    ud = torch.from_numpy(up).to(cuda).to(dt)
    g = qfb.fake_quantize_backward(xd, ls.tolist(), None, ud)
    _, dx, dls = orc.fq_backward(x, up, ls, 1, C, H * W)
    got = host(g.d_input.float()).ravel()
    assert np.array_equal(bits32(got), bits32(dx))
    check_grads(g.d_log_scale, dls, TOL_F16 if half else TOL_F32)


@pytest.mark.parametrize("half", [0, 1])
@pytest.mark.parametrize("which", ["x", "up", "dx"])
def test_unaligned_buffers(qfb, orc, cuda, half, which):
    """x, upstream or d_input starting off a 16-byte boundary (one element
    past an aligned allocation): the producer fills the stage itself and
    d_input is stored element-wise; results bitwise as on aligned buffers."""
    import torch
    rng = np.random.default_rng(31 + half)
    C, HW = 6, 4099
    n = C * HW
    x = rng.normal(0, 2, n).astype(np.float32)
    up = rng.normal(0, 1, n).astype(np.float32)
    if half:
        x = x.astype(np.float16).astype(np.float32)
        up = up.astype(np.float16).astype(np.float32)
    dt = torch.float16 if half else torch.float32
    ls = rng.uniform(-4, -1, C)

    def buf(a, off):
        base = torch.zeros(a.size + 8, dtype=dt, device=cuda)
        v = base[off:off + a.size]
        v.copy_(torch.from_numpy(a).to(dt))
        return base, v
    bx, xd = buf(x, 1 if which == "x" else 0)
    bu, ud = buf(up, 1 if which == "up" else 0)
    bd = torch.full((n + 8,), 7.0, dtype=dt, device=cuda)
    dxd = bd[1:1 + n] if which == "dx" else bd[:n]
    s64, chain = qfb.scale_grad_factors(ls.tolist())
    fac = torch.tensor(s64 + chain, dtype=torch.float64, device=cuda)
    dls = torch.zeros(C, dtype=torch.float64, device=cuda)
    ctx = qfb.default_context(0)
    code = qfb.F16 if half else qfb.F32
    qfb.check(qfb.lib().qfb_fq_bwd(ctx.handle, code, xd.data_ptr(), ud.data_ptr(), dxd.data_ptr(), 1, C, HW,
                                   fac.data_ptr(), fac.data_ptr() + 8 * C, 127, dls.data_ptr(), 0))
    ctx.sync()
    _, dx, want = orc.fq_backward(x, up, ls, 1, C, HW)
    assert np.array_equal(bits32(host(dxd.float())), bits32(dx))
    # the guard elements around d_input are untouched
    g = host(bd.float())
    lo = 1 if which == "dx" else 0
    assert np.all(g[:lo] == 7.0) and np.all(g[lo + n:] == 7.0)
    check_grads(dls.cpu().numpy(), want, TOL_F16 if half else TOL_F32)


def test_scales_outside_fast_range(qfb, orc, cuda):
    """Scales below 2^-100 or above 2^100 (reachable with a permissive
    QuantConfig: eps 0, s_min 1e-300, s_max 1e300) take the checked path
    with the exact IEEE quotient; per channel, every row long enough for
    9/10-element leaf groups. d_input and d_log_s bitwise."""
    import oracle as O
    rng = np.random.default_rng(41)
    C, HW = 4, 5000
    cfg = qfb.QuantConfig(eps=0.0, s_min=1e-300, s_max=1e300)
    ocfg = O.OrcCfg(8, 0, 1e-300, 1e-4, 1e300, 0.0)
    ls = np.array([-300.0, -240.0, 1e31, 1.5])   # s ~ 5e-131, 6e-105, 1e31, 1.7
    x = rng.normal(0, 1, (C, HW)).astype(np.float32)
    x[0, ::7] = 0.0
    x[1, ::5] = np.float32(1e-40)                # subnormal
    x[3] *= 2.0
    up = rng.normal(0, 1, (C, HW)).astype(np.float32)
    g = qfb.fake_quantize_backward(to_dev(x, cuda), ls.tolist(), cfg, to_dev(up, cuda))
    _, dx, dls = orc.fq_backward(x, up, ls, 1, C, HW, cfg=ocfg)
    assert np.array_equal(bits32(host(g.d_input).ravel()), bits32(dx))
    assert np.asarray(g.d_log_scale).tobytes() == dls.tobytes()


@pytest.mark.parametrize("n", [128 * 120 * 160, 11_000_000])
def test_long_rows_finisher_paths(qfb, orc, cuda, n):
    """Per-tensor backward over one long row: 2.46 M elements (config 1's
    map: 1,024 tiles per row -> the shared-memory finisher) and 11 M
    elements (> 4,096 tiles -> its in-place global path). d_input and
    d_log_s bitwise."""
    rng = np.random.default_rng(n % 1000)
    x = rng.normal(0, 1, n).astype(np.float32)
    up = rng.normal(0, 1, n).astype(np.float32)
    ls = -3.2
    g = qfb.fake_quantize_backward(to_dev(x, cuda), ls, None, to_dev(up, cuda))
    _, dx, dls = orc.fq_backward(x, up, [ls], 1, 1, n)
    assert np.array_equal(bits32(host(g.d_input)), bits32(dx))
    check_grads(g.d_log_scale, dls, TOL_F32)
