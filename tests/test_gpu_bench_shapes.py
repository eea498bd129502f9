"""The launch shapes the benchmark times, at their full sizes, against the
CPU oracle:

* config 5's forward: FrontendQuantPass(frames=8) at 480x640, f32 / f16,
  fake-quant values and int8 codes. For f32 this launch takes the 4-stage
  TMA ring (ew_tma_kernel<float, false, 4>, tma_stages() >= 64 chunks per
  CTA); every element is checked against 8 one-frame launches of the same
  frames (which the oracle pins in test_gpu_frontend.py), and frames 0 and 7
  against the oracle directly.
* the 4-stage ring forced (QFB_FWD_STAGES=4) on small tables, bitwise
  against the oracle.
* config 4's backward: the 64-frame QatStep at full size (outer = 64 rows
  per channel): its per-frame scale-gradient rows equal one-frame launches
  of the same frames bitwise, frames 0 and 63 equal the oracle, and the
  frame-order fold of the rows equals the oracle's accumulation.
Frame data depends only on the global frame index (frame_offset), so a
frame is the same bytes in every launch shape.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def b32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("int8_out", [False, True])
def test_c5_eight_frame_forward_full_size(qfb, orc, cuda, dtype, int8_out):
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    F, seed = 8, 31
    ctx = qfb.default_context(0)
    fp = FrontendQuantPass(ctx, frames=F, dtype=dtype, sets=1, seed=seed, device=cuda, int8_out=int8_out)
    fp.forward(0)
    torch.cuda.synchronize()
    ctx.sync()
    big = [y.cpu() for y in fp.y]
    log_s = fp.log_s
    del fp
    torch.cuda.empty_cache()
    # every frame against a one-frame launch of the same frame
    for f in range(F):
        one = FrontendQuantPass(ctx, frames=1, dtype=dtype, sets=1, seed=seed, device=cuda, int8_out=int8_out,
                                frame_offset=f)
        one.forward(0)
        torch.cuda.synchronize()
        for ci, y in enumerate(one.y):
            a = big[ci][f].numpy().ravel().view(np.uint8)
            b = y[0].cpu().numpy().ravel().view(np.uint8)
            assert np.array_equal(a, b), (f, one.consumers[ci][0].name)
        del one
        torch.cuda.empty_cache()
    # frames 0 and F-1 against the oracle
    half = 1 if dtype == "f16" else 0
    probe = FrontendQuantPass(ctx, frames=1, dtype=dtype, sets=1, seed=seed, device=cuda, int8_out=int8_out)
    for f in (0, F - 1):
        ci = 0
        for pi, p in enumerate(probe.points):
            x = orc.fill_rng(p.numel, seed, pi, kind=1, lo=1.0, offset=f * p.numel, half=half)
            for _k in p.consumers:
                s64 = np.array(qfb.scale_grad_factors(log_s[ci].tolist())[0])
                got = big[ci][f].numpy().ravel()
                if int8_out:
                    _, want = orc.int8_codes(x, s64, 1, p.channels, p.inner)
                    assert np.array_equal(got, want), (f, p.name)
                else:
                    _, want = orc.fake_quantize(x, s64, 1, p.channels, p.inner, half=half)
                    assert np.array_equal(b32(got.astype(np.float32)), b32(want)), (f, p.name)
                ci += 1


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_forced_four_stage_ring(qfb, orc, cuda, dtype, monkeypatch):
    """QFB_FWD_STAGES=4 (read at context creation) on a table of small
    points: the 4-stage TMA ring, bitwise against the oracle."""
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    monkeypatch.setenv("QFB_FWD_STAGES", "4")
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    F, h, w = 3, 64, 96
    half = 1 if dtype == "f16" else 0
    fp = FrontendQuantPass(ctx, frames=F, dtype=dtype, sets=1, seed=13, device=cuda, h=h, w=w)
    fp.forward(0)
    ctx.sync()
    ci = 0
    for pi, p in enumerate(fp.points):
        x = orc.fill_rng(F * p.numel, 13, pi, kind=1, lo=1.0, half=half)
        for _k in p.consumers:
            s64 = np.array(qfb.scale_grad_factors(fp.log_s[ci].tolist())[0])
            _, want = orc.fake_quantize(x, s64, F, p.channels, p.inner, half=half)
            assert np.array_equal(b32(fp.y[ci].float().cpu().numpy().ravel()), b32(want)), p.name
            ci += 1
    ctx.close()
    monkeypatch.delenv("QFB_FWD_STAGES")


def test_c4_sixty_four_frame_backward_full_size(qfb, orc, cuda):
    """The config-4 launch (64 frames of 480x640 per launch): rows of the
    64-frame backward vs one-frame launches, the oracle on frames 0 and 63,
    and the fold of all rows vs the oracle's frame-order accumulation
    (computed from the one-frame rows the oracle pinned)."""
    import torch
    from paper_2511_12653_b200.frontend import QatStep
    F, seed = 64, 23
    ctx = qfb.default_context(0)
    qs = QatStep(ctx, frames=F, seed=seed, device=cuda)
    qs.resolve_scales()
    qs.forward_backward()
    qs.exchange()
    ctx.sync()
    rows = qs.rows.cpu().numpy()
    folded = qs.grads[:qs.n_act].cpu().numpy()
    log_s = [ls.copy() for ls in qs.fp.log_s]
    points = qs.fp.points
    del qs
    torch.cuda.empty_cache()
    # one-frame launches of the same frames (frame_offset), rows mode
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    n_grad = rows.shape[1]
    for f in range(F):
        r1 = torch.zeros((1, n_grad), dtype=torch.float64, device=cuda)
        one = FrontendQuantPass(ctx, frames=1, sets=1, seed=seed, device=cuda, rows_out=r1, frame_offset=f)
        one.backward(0)
        ctx.sync()
        assert r1.cpu().numpy()[0].tobytes() == rows[f].tobytes(), f
        del one
    torch.cuda.empty_cache()
    # frames 0 and 63 against the oracle (chain-scaled per-row results)
    for f in (0, F - 1):
        ci, goff = 0, 0
        for pi, p in enumerate(points):
            x = orc.fill_rng(p.numel, seed, pi, kind=1, lo=1.0, offset=f * p.numel)
            for _k in p.consumers:
                up = orc.fill_rng(p.numel, seed + 500, ci, kind=1, lo=1.0, offset=f * p.numel)
                _, _, dls = orc.fq_backward(x, up, log_s[ci], 1, p.channels, p.inner, want_dx=False)
                assert rows[f, goff:goff + p.channels].tobytes() == dls.tobytes(), (f, p.name)
                goff += p.channels
                ci += 1
    # the frame-order fold ((r0 + r1) + ...) of the rows
    acc = rows[0].copy()
    for f in range(1, F):
        acc = acc + rows[f]
    assert folded.tobytes() == acc.tobytes()
