"""GPU parity for the QAT-step pieces through the C-ABI:
qfb_distill_pair / distill_loss (bitwise vs the oracle and vs the
reference-made vectors, including DPVO fnet/inet output sizes) and
qfb_adam_step (bitwise vs the oracle, skip on a non-finite gradient)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "distill_vectors.npz")


def b32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def dev(a, cuda):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def test_golden_vectors_on_device(qfb, cuda):
    g = np.load(GOLD)
    for k in range(int(g["n_cases"])):
        lam = float(g[f"lam{k}"])
        res, df, di = qfb.distill_loss(dev(g[f"fs{k}"], cuda), dev(g[f"ft{k}"], cuda), dev(g[f"is{k}"], cuda),
                                       dev(g[f"it{k}"], cuda), lam)
        got = np.array([res["total"], res["mse_f"], res["mse_i"], res["cos_f"], res["cos_i"]])
        assert got.tobytes() == g[f"out{k}"].tobytes(), (k, got, g[f"out{k}"])
        assert np.array_equal(b32(df.cpu().numpy()), b32(g[f"df{k}"]))
        assert np.array_equal(b32(di.cpu().numpy()), b32(g[f"di{k}"]))


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 1, 1), (3, 17, 9), (128, 120, 160), (384, 120, 160),
                                   (64, 1, 4097)])
@pytest.mark.parametrize("grad_scale", [1.0, 1.0 / 15])
def test_pair_vs_oracle(qfb, orc, cuda, shape, grad_scale):
    rng = np.random.default_rng(sum(shape))
    s, t = [rng.normal(0, 1, shape).astype(np.float32) for _ in range(2)]
    s.reshape(shape[0], -1)[:, ::97] = 0.0   # zero-norm locations
    st, o2, ds = orc.distill_pair(s, t, 0.9, grad_scale)
    d, out2 = qfb.distill_pair(dev(s, cuda), dev(t, cuda), 0.9, grad_scale)
    assert out2.cpu().numpy().tobytes() == o2.tobytes()
    assert np.array_equal(b32(d.cpu().numpy()), b32(ds))


def test_adam_vs_oracle_and_skip(qfb, orc, cuda):
    import torch
    rng = np.random.default_rng(12)
    n = 1494                       # the DPVO scale-parameter count
    p = rng.normal(-3, 1, n)
    m = np.zeros(n)
    v = np.zeros(n)
    P, M, V = dev(p, cuda), dev(m, cuda), dev(v, cuda)
    for t in range(1, 6):
        g = rng.normal(0, 1e-2, n)
        assert orc.adam(p, m, v, g, 0.9, 0.999, 5e-3, 1e-8, t) == 0
        sk = qfb.adam_step(P, M, V, dev(g, cuda), t, 5e-3)
        assert int(sk.item()) == 0
        assert P.cpu().numpy().tobytes() == p.tobytes()
        assert M.cpu().numpy().tobytes() == m.tobytes() and V.cpu().numpy().tobytes() == v.tobytes()
    g = rng.normal(0, 1e-2, n)
    g[100] = np.inf
    before = P.clone()
    sk = qfb.adam_step(P, M, V, dev(g, cuda), 6, 5e-3)
    torch.cuda.synchronize()
    assert int(sk.item()) == 1 and torch.equal(P, before)


def test_fold_rows_device_is_frame_order(qfb, cuda):
    """qfb_fold_rows == ((into + r0) + r1) + ... bit for bit (the exchange's
    combine step, dist.fold_rows on CUDA tensors)."""
    import torch
    from paper_2511_12653_b200.dist import fold_rows
    rng = np.random.default_rng(3)
    rows = rng.normal(0, 1, (8, 1494)) * np.exp(rng.uniform(-30, 30, (8, 1494)))
    into = rng.normal(0, 1, 1494)
    want = rows[0].copy()
    for r in rows[1:]:
        want = want + r
    want2 = into + rows[0]
    for r in rows[1:]:
        want2 = want2 + r
    got = fold_rows(dev(rows, cuda))
    got2 = fold_rows(dev(rows, cuda), into=dev(into, cuda))
    torch.cuda.synchronize()
    assert got.cpu().numpy().tobytes() == want.tobytes()
    assert got2.cpu().numpy().tobytes() == want2.tobytes()


def test_context_teardown_frees_device_memory(qfb, cuda):
    """Contexts that ran the trainer ops (their scratch) and the backward are
    destroyed without leaking device memory (qfb_ctx_destroy frees every
    workspace after synchronizing its streams)."""
    import torch
    s = torch.randn((128, 120, 160), device=cuda)
    t = torch.randn_like(s)
    x = torch.randn((64, 120, 160), device=cuda)
    up = torch.randn_like(x)

    def cycle():
        ctx = qfb.Context(0)
        qfb.distill_pair(s, t, 1.0, ctx=ctx)
        qfb.fake_quantize_backward(x, [-3.0] * 64, None, up, ctx=ctx)
        ctx.sync()
        ctx.close()

    cycle()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(10):
        cycle()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 8 << 20, (free0, free1)
