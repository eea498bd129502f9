"""The opt-in float32-term backward for binary16 storage
(QFB_OPT_BWD_HALF_FP32): d_input must stay bit-identical to the oracle (the
clip mask is decided exactly through the per-tile binary16 threshold), the
scale gradients must meet north_star's FP16 tolerance (rel 1e-2) — asserted
here much tighter: |err| <= 1e-5 |ref| + 2^-20 sum|terms|, the float32
rounding of each term and of the 9..16-term leaf folds — and the option off
must give the exact (bitwise) path back. Rows: full-tile lengths (the fast
path) and short ones (the exact fallback), specials, values on and half-way
between quantization levels, a clamp-gated channel, frames as outer rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LENGTHS = [2048, 4104, 8200, 19200, 65544, 76800, 307200]


def inputs(n, C, outer, seed):
    rng = np.random.default_rng(seed)
    s64 = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
    x = (rng.normal(0, 1, (outer, C, n)) * (s64[None, :, None] * 90)).astype(np.float16).astype(np.float32)
    up = rng.normal(0, 1, (outer, C, n)).astype(np.float16).astype(np.float32)
    fx, fu = x.reshape(-1), up.reshape(-1)
    k = rng.integers(0, fx.size, 64)
    fx[k[:6]] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 65504.0]
    fu[k[8:12]] = [0.0, -0.0, 65504.0, -65504.0]
    # exactly on the grid and exactly half-way between codes (binary16 values)
    fx[k[16:40]] = ((rng.integers(-140, 140, 24) * 0.5) * s64[0]).astype(np.float16).astype(np.float32)
    chain = 1.0 / (1.0 + np.exp(-np.log(np.expm1(s64))))
    chain[-1] = 0.0
    return x, up, s64, chain


def abs_terms(x, up, s64, outer, C, n):
    """sum |d_ds * up| per channel (binary64, numpy IEEE division)."""
    z = x.reshape(outer, C, n).astype(np.float64) / s64[None, :, None]
    u = up.reshape(outer, C, n).astype(np.float64)
    with np.errstate(invalid="ignore"):
        mask = np.abs(z) <= 127.0
        d = np.where(mask, np.rint(z) - z, np.where(z > 0, 127.0, -127.0))
        t = np.abs(d * u)
    return np.nansum(np.where(np.isfinite(t), t, 0.0), axis=(0, 2))


def run(qfb, cuda, ctx, x, up, s64, chain, outer, C, n):
    import torch
    xd = torch.from_numpy(x).to(cuda).to(torch.float16)
    ud = torch.from_numpy(up).to(cuda).to(torch.float16)
    dx = torch.empty_like(xd)
    fac = torch.tensor(np.concatenate([s64, chain]), dtype=torch.float64, device=cuda)
    dls = torch.zeros(C, dtype=torch.float64, device=cuda)
    qfb.check(qfb.lib().qfb_fq_bwd(ctx.handle, 1, xd.data_ptr(), ud.data_ptr(), dx.data_ptr(), outer, C, n,
                                   fac.data_ptr(), fac.data_ptr() + 8 * C, 127, dls.data_ptr(), 0))
    ctx.sync()
    return dx.float().cpu().numpy().ravel(), dls.cpu().numpy()


@pytest.mark.parametrize("n", LENGTHS)
def test_half_fp32_terms_within_tolerance(qfb, orc, cuda, n):
    C, outer = 3, 2
    x, up, s64, chain = inputs(n, C, outer, 100 + n)
    ctx = qfb.Context(0)
    ctx.set_option(qfb.OPT_BWD_HALF_FP32, 1)
    dx, dls = run(qfb, cuda, ctx, x, up, s64, chain, outer, C, n)
    _, dx_o, dls_o = orc.fq_backward_s(x, up, s64, chain, outer, C, n)
    nan = np.isnan(dx_o)
    assert np.array_equal(np.isnan(dx), nan)
    assert np.array_equal(dx[~nan].view(np.uint32), dx_o[~nan].view(np.uint32))
    fin = ~np.isnan(dls_o)
    assert np.array_equal(np.isnan(dls), ~fin)
    bound = 1e-5 * np.abs(dls_o) + 2.0 ** -20 * abs_terms(x, up, s64, outer, C, n) * np.abs(chain)
    err = np.abs(dls - dls_o)
    assert np.all(err[fin] <= bound[fin]), (err, bound)
    # north_star's FP16 tolerance holds with room to spare
    ok = fin & (np.abs(dls_o) > 0)
    assert np.all(err[ok] <= 1e-2 * np.abs(dls_o[ok]))
    ctx.close()


def test_option_off_is_bitwise_and_validated(qfb, orc, cuda):
    n, C, outer = 76800, 2, 1
    x, up, s64, chain = inputs(n, C, outer, 7)
    ctx = qfb.Context(0)
    ctx.set_option(qfb.OPT_BWD_HALF_FP32, 1)
    ctx.set_option(qfb.OPT_BWD_HALF_FP32, 0)
    dx, dls = run(qfb, cuda, ctx, x, up, s64, chain, outer, C, n)
    _, dx_o, dls_o = orc.fq_backward_s(x, up, s64, chain, outer, C, n)
    fin = ~np.isnan(dls_o)
    assert dls[fin].tobytes() == dls_o[fin].tobytes()
    with pytest.raises(qfb.ValueError):
        ctx.set_option(qfb.OPT_BWD_HALF_FP32, 2)
    with pytest.raises(qfb.ValueError):
        ctx.set_option(99, 1)
    ctx.close()


def test_f32_storage_ignores_the_option(qfb, orc, cuda):
    """The option concerns binary16 storage only: f32 stays bitwise."""
    import torch
    n, C, outer = 19200, 2, 2
    rng = np.random.default_rng(3)
    s64 = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
    x = (rng.normal(0, 1, (outer, C, n)) * (s64[None, :, None] * 90)).astype(np.float32)
    up = rng.normal(0, 1, (outer, C, n)).astype(np.float32)
    chain = np.full(C, 0.5)
    ctx = qfb.Context(0)
    ctx.set_option(qfb.OPT_BWD_HALF_FP32, 1)
    xd, ud = torch.from_numpy(x).to(cuda), torch.from_numpy(up).to(cuda)
    dx = torch.empty_like(xd)
    fac = torch.tensor(np.concatenate([s64, chain]), dtype=torch.float64, device=cuda)
    dls = torch.zeros(C, dtype=torch.float64, device=cuda)
    qfb.check(qfb.lib().qfb_fq_bwd(ctx.handle, 0, xd.data_ptr(), ud.data_ptr(), dx.data_ptr(), outer, C, n,
                                   fac.data_ptr(), fac.data_ptr() + 8 * C, 127, dls.data_ptr(), 0))
    ctx.sync()
    _, dx_o, dls_o = orc.fq_backward_s(x, up, s64, chain, outer, C, n)
    assert np.array_equal(dx.cpu().numpy().ravel().view(np.uint32), dx_o.view(np.uint32))
    assert dls.cpu().numpy().tobytes() == dls_o.tobytes()
    ctx.close()
