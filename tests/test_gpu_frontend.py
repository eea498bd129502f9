"""The benchmarked workloads themselves against the CPU oracle: every
output of FrontendQuantPass (config 2: 22 quant points, multi-consumer
points, frames as rows, f32 / f16 storage, FQ values or int8 codes) and of
WindowChainPass (config 3 chains: residual joins, ReLU / GELU, patch and
update-operator points), at reduced frame sizes with the same structure."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def b32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("int8_out", [False, True])
def test_frontend_pass_matches_oracle(qfb, orc, cuda, dtype, int8_out):
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    F, h, w = 2, 48, 64
    ctx = qfb.default_context(0)
    fp = FrontendQuantPass(ctx, frames=F, dtype=dtype, sets=2, seed=5, device=cuda, h=h, w=w,
                           int8_out=int8_out)
    half = 1 if dtype == "f16" else 0
    for si in range(2):
        fp.forward(si)
        fp.backward(si)
        torch.cuda.synchronize()
        ctx.sync()
        ci = 0
        for pi, p in enumerate(fp.points):
            n = F * p.numel
            x = orc.fill_rng(n, 5 + 1000 * si, pi, kind=1, lo=1.0, half=half)
            for k in range(len(p.consumers)):
                up = orc.fill_rng(n, 5 + 1000 * si + 500, ci, kind=1, lo=1.0, half=half)
                s64 = np.array(qfb.scale_grad_factors(fp.log_s[ci].tolist())[0])
                if int8_out:
                    _, want = orc.int8_codes(x, s64, F, p.channels, p.inner)
                    assert np.array_equal(fp.y[ci].cpu().numpy().ravel(), want), (p.name, k)
                else:
                    _, want = orc.fake_quantize(x, s64, F, p.channels, p.inner, half=half)
                    got = fp.y[ci].float().cpu().numpy().ravel()
                    assert np.array_equal(b32(got), b32(want)), (p.name, k)
                # factors are Full-mode (FrontendQuantPass resolves them so); the values are
                # already on the binary16 grid for f16 storage
                _, dx, dls = orc.fq_backward(x, up, fp.log_s[ci], F, p.channels, p.inner)
                assert np.array_equal(b32(fp.dx[ci].float().cpu().numpy().ravel()), b32(dx)), (p.name, k)
                assert fp.dls[ci].cpu().numpy().tobytes() == dls.tobytes(), (p.name, k)
                ci += 1


@pytest.mark.parametrize("dtype,full", [("f32", False), ("f32", True), ("f16", False), ("f16", True)])
@pytest.mark.parametrize("gelu", [False, True])
def test_window_chain_pass_matches_oracle(qfb, orc, cuda, gelu, dtype, full):
    """full=True is BASELINE config 3 as benched (15-frame window, 96 patches,
    480x640); f16 stores a, b and the outputs in binary16 (the oracle gets
    the same half-grid values as float, half=1)."""
    import torch
    from paper_2511_12653_b200.frontend import WindowChainPass
    ctx = qfb.default_context(0)
    if full:
        wp = WindowChainPass(ctx, gelu=gelu, dtype=dtype, device=cuda)
    else:
        wp = WindowChainPass(ctx, frames=2, patches=4, gelu=gelu, dtype=dtype, device=cuda, h=48, w=64)
    wp.run()
    torch.cuda.synchronize()
    ctx.sync()
    half = 1 if dtype == "f16" else 0
    for p, (a, b, ys, ss) in zip(wp.points, wp.buffers):
        ah = a.float().cpu().numpy()
        bh = b.float().cpu().numpy() if b is not None else None
        scales = [np.asarray(s, dtype=np.float64) for s in ss]
        st, want, _ = orc.fq_chain(ah, bh, scales, p.outer, p.channels, p.inner, act=p.act, half=half)
        assert st == 0
        for y, w in zip(ys, want):
            assert np.array_equal(b32(y.float().cpu().numpy()), b32(w)), p.name


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_full_size_frame_matches_oracle(qfb, orc, cuda, dtype):
    """BASELINE config 2 at full size (one 480x640 frame, 41.2 M quant-point
    elements): every forward output, d_input and scale gradient of the
    benchmarked pass equals the oracle, plus a size-independent property
    (FQ values sit on their channel's grid s*q, |q| <= 128)."""
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    ctx = qfb.default_context(0)
    fp = FrontendQuantPass(ctx, frames=1, dtype=dtype, sets=1, seed=77, device=cuda)
    half = 1 if dtype == "f16" else 0
    fp.forward(0)
    fp.backward(0)
    torch.cuda.synchronize()
    ctx.sync()
    ci = 0
    for pi, p in enumerate(fp.points):
        x = orc.fill_rng(p.numel, 77, pi, kind=1, lo=1.0, half=half)
        for _k in p.consumers:
            s64 = np.array(qfb.scale_grad_factors(fp.log_s[ci].tolist())[0])
            _, want = orc.fake_quantize(x, s64, 1, p.channels, p.inner, half=half)
            got = fp.y[ci].float().cpu().numpy().ravel()
            assert np.array_equal(b32(got), b32(want)), p.name
            codes = got.astype(np.float64).reshape(p.channels, -1) / s64[:, None]
            tol = 1e-3 if half else 1e-6
            assert np.all(np.abs(codes - np.rint(codes)) <= tol * np.maximum(1.0, np.abs(codes)))
            assert np.all(np.abs(np.rint(codes)) <= 128)
            up = orc.fill_rng(p.numel, 77 + 500, ci, kind=1, lo=1.0, half=half)
            _, dx, dls = orc.fq_backward(x, up, fp.log_s[ci], 1, p.channels, p.inner)
            assert np.array_equal(b32(fp.dx[ci].float().cpu().numpy().ravel()), b32(dx)), p.name
            assert fp.dls[ci].cpu().numpy().tobytes() == dls.tobytes(), p.name
            ci += 1
