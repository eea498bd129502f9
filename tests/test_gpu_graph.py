"""The device entry points are CUDA-graph capturable: descriptor tables
travel as kernel parameters, workspaces are sized on first use, the
backward finisher is stateless. A captured fwd+bwd step replays bit-exactly."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_frontend_step_graph_replay(qfb, cuda):
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    fp = FrontendQuantPass(ctx, frames=2, dtype="f32", sets=1, h=48, w=64, device=cuda)
    with torch.cuda.stream(stream):
        fp.forward(0)
        fp.backward(0)
    ctx.sync()
    y_ref = [t.clone() for t in fp.y]
    dx_ref = [t.clone() for t in fp.dx]
    g_ref = fp.scale_grads().clone()
    for t in fp.y + fp.dx + fp.dls:
        t.zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fp.forward(0)
        fp.backward(0)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ctx.sync()
    for a, b in zip(fp.y, y_ref):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    for a, b in zip(fp.dx, dx_ref):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    assert torch.equal(fp.scale_grads().view(torch.int64), g_ref.view(torch.int64))
    ctx.close()


def _bwd(qfb, ctx, x, up, dx, fac, dls, C, inner):
    return qfb.lib().qfb_fq_bwd(ctx.handle, 0, x.data_ptr(), up.data_ptr(), dx.data_ptr(), 1, C, inner,
                                fac.data_ptr(), fac.data_ptr() + 8 * C, 127, dls.data_ptr(), 0)


def test_captured_backward_survives_workspace_growth(qfb, cuda):
    """A graph captured with a small backward keeps its workspace after a
    larger eager backward grows the context's (the old buffer is retired,
    not freed): replays stay bitwise identical (run under compute-sanitizer
    memcheck by tools/gpu_sanitize_r02.sh)."""
    import torch
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)

    def make(C, inner, seed):
        x = torch.empty(C * inner, device=cuda)
        up = torch.empty(C * inner, device=cuda)
        qfb.fill_rng(x, seed=seed, stream=0, ctx=ctx)
        qfb.fill_rng(up, seed=seed, stream=1, ctx=ctx)
        ls = np.log(np.expm1(np.exp(np.random.default_rng(seed).uniform(np.log(1e-3), np.log(0.1), C))))
        s64, chain = qfb.scale_grad_factors(ls.tolist())
        fac = torch.tensor(s64 + chain, dtype=torch.float64, device=cuda)
        return x, up, torch.empty_like(x), fac, torch.zeros(C, dtype=torch.float64, device=cuda)

    C, n = 4, 5000
    small = make(C, n, 3)
    qfb.check(_bwd(qfb, ctx, *small, C, n))  # eager: sizes the workspace for this shape
    ctx.sync()
    want_dx, want_g = small[2].clone(), small[4].clone()
    small[2].zero_()
    small[4].zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        qfb.check(_bwd(qfb, ctx, *small, C, n))
    g.replay()
    ctx.sync()
    assert torch.equal(small[4], want_g)
    # a much larger backward on the same context grows the workspace
    Cb, nb = 64, 300000
    big = make(Cb, nb, 4)
    qfb.check(_bwd(qfb, ctx, *big, Cb, nb))
    ctx.sync()
    small[2].zero_()
    small[4].zero_()
    torch.cuda.synchronize()
    for _ in range(2):
        g.replay()
    ctx.sync()
    assert torch.equal(small[2].view(torch.int32), want_dx.view(torch.int32))
    assert torch.equal(small[4].view(torch.int64), want_g.view(torch.int64))
    ctx.close()


def test_growth_under_capture_is_refused(qfb, cuda):
    """A first (unsized) backward inside a stream capture returns
    QFB_ERR_UNSUPPORTED before enqueueing anything; after
    qfb_fq_bwd_reserve the same call captures and replays."""
    import torch
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    C, n = 8, 40000
    x = torch.empty(C * n, device=cuda)
    up = torch.empty(C * n, device=cuda)
    qfb.fill_rng(x, seed=5, stream=0, ctx=ctx)
    qfb.fill_rng(up, seed=5, stream=1, ctx=ctx)
    s64, chain = qfb.scale_grad_factors([-4.0] * C)
    fac = torch.tensor(s64 + chain, dtype=torch.float64, device=cuda)
    dx = torch.empty_like(x)
    dls = torch.zeros(C, dtype=torch.float64, device=cuda)
    ctx.sync()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        st = _bwd(qfb, ctx, x, up, dx, fac, dls, C, n)
    assert st == 9  # QFB_ERR_UNSUPPORTED
    d = qfb.CBwdDesc()
    d.x, d.up, d.dx = x.data_ptr(), up.data_ptr(), dx.data_ptr()
    d.scale64, d.chain, d.d_log_s = fac.data_ptr(), fac.data_ptr() + 8 * C, dls.data_ptr()
    d.outer, d.channels, d.inner, d.q_max, d.accumulate = 1, C, n, 127, 0
    qfb.check(qfb.lib().qfb_fq_bwd_reserve(ctx.handle, 0, ctypes.byref(d), 1))
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=stream):
        qfb.check(_bwd(qfb, ctx, x, up, dx, fac, dls, C, n))
    g2.replay()
    ctx.sync()
    want = qfb.fake_quantize_backward(x.view(C, n), [-4.0] * C, None, up.view(C, n))
    assert dls.cpu().tolist() == want.d_log_scale
    ctx.close()
