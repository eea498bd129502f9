"""BASELINE config 4 pieces composed (frontend.QatStep, reduced frame
size): per-frame distillation loss and its scaled gradients, the scale-only
backward's frame-ordered gradients landing in the optimizer vector, and the
Adam update — each bitwise against the oracle composition."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_qat_step_matches_oracle(qfb, orc, cuda):
    import torch
    from paper_2511_12653_b200.frontend import QatStep
    F = 3
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    qs = QatStep(ctx, frames=F, seed=9, device=cuda, h=32, w=64)
    p0 = qs.params.cpu().numpy().copy()
    with torch.cuda.stream(stream):
        qs.run()
    stream.synchronize()
    ctx.sync()
    # distillation: loss values and gradients per frame and pair
    loss = qs.losses()
    for f in range(F):
        for k, (c, s, t, d) in enumerate(qs.feat):
            st, o2, ds = orc.distill_pair(s[f].cpu().numpy(), t[f].cpu().numpy(), qs.lam, 1.0 / F)
            assert st == 0
            assert loss[f, k].cpu().numpy().tobytes() == o2.tobytes()
            assert np.array_equal(d[f].cpu().numpy().view(np.uint32), ds.view(np.uint32))
    # scale gradients: consumer order, rows (frames) accumulated in order
    fp = qs.fp
    g = []
    ci = 0
    for pi, p in enumerate(fp.points):
        x = orc.fill_rng(F * p.numel, 9, pi, kind=1, lo=1.0)
        for _k in p.consumers:
            up = orc.fill_rng(F * p.numel, 9 + 500, ci, kind=1, lo=1.0)
            _, _, dls = orc.fq_backward(x, up, fp.log_s[ci], F, p.channels, p.inner, want_dx=False)
            g.append(dls)
            ci += 1
    g = np.concatenate(g + [np.zeros(qs.n_params - qs.n_act)])
    assert qs.grads.cpu().numpy().tobytes() == g.tobytes()
    # Adam on the whole vector
    m = np.zeros_like(p0)
    v = np.zeros_like(p0)
    assert orc.adam(p0, m, v, g, 0.9, 0.999, qs.lr, 1e-8, 1) == 0
    assert qs.params.cpu().numpy().tobytes() == p0.tobytes()
    assert int(qs.skipped.item()) == 0
    ctx.close()
