"""Every backward kernel variant against the CPU oracle, bitwise: the tile
kernel with consumer-side warp partials (default), the round-1 tile kernel
(QFB_BWD_IMPL=tile1) and the streaming kernel (QFB_BWD_IMPL=stream: fixed
row chunks, chunk-owned tree blocks of 16 leaf groups). Row lengths
around the chunk and block bounds, f32 and f16 storage, frames as outer
rows, specials (NaN / inf in x and upstream, signed zeros, saturated and
exactly-on-the-grid values), a scale below 2^-100 (the exact slow path)
and a clamp-gated channel; one DPVO-shaped table through all three gives
the same bits."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LENGTHS = [2048, 2056, 2304, 4096, 4104, 6144, 8200, 12288, 19200, 65544, 76800, 100000, 123456, 307200]


def run(qfb, cuda, x, up, s64, chain, outer, C, n, dtype, ctx):
    import torch
    tdt = torch.float32 if dtype == 0 else torch.float16
    xd = torch.from_numpy(x).to(cuda).to(tdt)
    ud = torch.from_numpy(up).to(cuda).to(tdt)
    dx = torch.empty_like(xd)
    fac = torch.tensor(np.concatenate([s64, chain]), dtype=torch.float64, device=cuda)
    dls = torch.zeros(C, dtype=torch.float64, device=cuda)
    qfb.check(qfb.lib().qfb_fq_bwd(ctx.handle, dtype, xd.data_ptr(), ud.data_ptr(), dx.data_ptr(), outer, C, n,
                                   fac.data_ptr(), fac.data_ptr() + 8 * C, 127, dls.data_ptr(), 0))
    ctx.sync()
    return dx.float().cpu().numpy().ravel(), dls.cpu().numpy()


def inputs(n, C, outer, dtype, seed):
    rng = np.random.default_rng(seed)
    s64 = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
    x = (rng.normal(0, 1, (outer, C, n)) * (s64[None, :, None] * 90)).astype(np.float32)
    up = rng.normal(0, 1, (outer, C, n)).astype(np.float32)
    flat_x, flat_u = x.reshape(-1), up.reshape(-1)
    k = rng.integers(0, flat_x.size, 64)
    flat_x[k[:8]] = [np.nan, -np.nan, np.inf, -np.inf, 0.0, -0.0, 1e30, -1e30]
    flat_u[k[8:14]] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 65504.0]
    # values exactly on the grid and half-way between codes
    flat_x[k[16:40]] = (rng.integers(-140, 140, 24) * 0.5).astype(np.float32) * np.float32(s64[0])
    if dtype == 1:
        x = x.astype(np.float16).astype(np.float32)
        up = up.astype(np.float16).astype(np.float32)
    chain = 1.0 / (1.0 + np.exp(-np.log(np.expm1(s64))))
    chain[-1] = 0.0  # clamp-gated channel
    return x, up, s64, chain


IMPLS = ["default", "stream", "tile1", "tile", "tilem", "tileq", "tileqmd", "tile2d", "tiledp", "tiledu"]


def make_ctx(qfb, impl, monkeypatch):
    if impl != "default":
        monkeypatch.setenv("QFB_BWD_IMPL", impl)
    ctx = qfb.Context(0)
    monkeypatch.delenv("QFB_BWD_IMPL", raising=False)
    return ctx


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("n", LENGTHS)
@pytest.mark.parametrize("outer", [1, 2])
def test_backward_variants_match_oracle(qfb, orc, cuda, n, dtype, impl, outer, monkeypatch):
    """outer = 1: rows complete inside the main pass (fused finish) on the
    full-tile kernels; outer = 2 (frames folded per channel): the finisher
    kernel."""
    if dtype == 1 and n % 8:
        pytest.skip("f16 rows must be 16-byte multiples")
    C = 3
    x, up, s64, chain = inputs(n, C, outer, dtype, n + dtype)
    ctx = make_ctx(qfb, impl, monkeypatch)
    dx, dls = run(qfb, cuda, x, up, s64, chain, outer, C, n, dtype, ctx)
    _, dx_o, dls_o = orc.fq_backward_s(x, up, s64, chain, outer, C, n)
    if dtype == 0:
        assert np.array_equal(dx.view(np.uint32), dx_o.view(np.uint32))
    else:
        # binary16 storage: NaN payloads are not representable bit for bit
        nan = np.isnan(dx_o)
        assert np.array_equal(np.isnan(dx), nan)
        assert np.array_equal(dx[~nan].view(np.uint32), dx_o[~nan].view(np.uint32))
    # a channel with NaN terms: NaN (the payload of a NaN sum is not part
    # of the contract; finite channels are bitwise)
    fin = ~np.isnan(dls_o)
    assert np.array_equal(np.isnan(dls), ~fin)
    assert dls[fin].tobytes() == dls_o[fin].tobytes()


@pytest.mark.parametrize("impl", IMPLS)
def test_unusable_scale_takes_exact_path(qfb, orc, cuda, impl, monkeypatch):
    n, C, outer = 8200, 2, 1
    x, up, s64, chain = inputs(n, C, outer, 0, 5)
    s64[0] = 1e-35          # below 2^-100: the IEEE-division slow path
    x[0, 0] *= 1e-30
    ctx = make_ctx(qfb, impl, monkeypatch)
    dx, dls = run(qfb, cuda, x, up, s64, chain, outer, C, n, 0, ctx)
    _, dx_o, dls_o = orc.fq_backward_s(x, up, s64, chain, outer, C, n)
    assert np.array_equal(dx.view(np.uint32), dx_o.view(np.uint32))
    assert dls.tobytes() == dls_o.tobytes()


@pytest.mark.parametrize("dtype", [0, 1])
def test_variants_agree_on_dpvo_table(qfb, cuda, dtype, monkeypatch):
    """One DPVO-shaped table (3 row lengths, frames as rows) through all the
    kernels: identical d_input and scale gradients."""
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    out = []
    for impl in IMPLS:
        if impl != "default":
            monkeypatch.setenv("QFB_BWD_IMPL", impl)
        stream = torch.cuda.Stream(device=cuda)
        ctx = qfb.Context(0, stream.cuda_stream)
        fp = FrontendQuantPass(ctx, frames=2, dtype="f32" if dtype == 0 else "f16", sets=1, seed=3, device=cuda,
                               h=240, w=320)
        fp.backward(0)
        ctx.sync()
        out.append(([t.cpu() for t in fp.dx], fp.scale_grads().cpu()))
        ctx.close()
        monkeypatch.delenv("QFB_BWD_IMPL", raising=False)
    # the default kernel with its tiles visited first to last (QFB_BWD_ORDER=fwd;
    # the default visits them last to first)
    monkeypatch.setenv("QFB_BWD_ORDER", "fwd")
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    fp = FrontendQuantPass(ctx, frames=2, dtype="f32" if dtype == 0 else "f16", sets=1, seed=3, device=cuda,
                           h=240, w=320)
    fp.backward(0)
    ctx.sync()
    out.append(([t.cpu() for t in fp.dx], fp.scale_grads().cpu()))
    ctx.close()
    monkeypatch.delenv("QFB_BWD_ORDER", raising=False)
    (dxa, ga) = out[0]
    for (dxb, gb) in out[1:]:
        assert torch.equal(ga.view(torch.int64), gb.view(torch.int64))
        for a, b in zip(dxa, dxb):
            assert torch.equal(a.view(torch.int16 if dtype else torch.int32),
                               b.view(torch.int16 if dtype else torch.int32))
