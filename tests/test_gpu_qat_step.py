"""BASELINE config 4 composed (frontend.QatStep, reduced frame size): the
per-frame distillation loss and its scaled gradients, the scale-only
backward's per-frame gradient rows and their frame-order fold into the
optimizer vector, and Adam with the step counter on the device — each
bitwise against the oracle composition, over several successive steps
(scales re-resolved from the updated log scales every step,
frontend.hpp:103-120; t = non-skipped steps, distill.hpp:262-264).

Multi-GPU semantics (distill.hpp:243-279 with the chunk's frames sharded):
two ranks holding frames [0, 2) and [2, 4) exchange their rows BEFORE Adam
and end the step with bitwise-equal replicas, equal to the one-process
4-frame step. On the one-GPU box the two ranks share cuda:0 and exchange
through gloo (NCCL refuses two ranks on one device); the NCCL C-ABI path
(qfb_nccl_comm_init_rank + qfb_gather_fold_scale_grads) is checked on a
one-rank communicator."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def oracle_step(orc, qs, p, m, v, t):
    """One step of the reference trainer restated on the oracle: scales from
    the current log scales p, per-frame rows, frame-order fold, Adam."""
    fp = qs.fp
    F = qs.frames
    g = []
    ci = 0
    off = 0
    for pi, pt in enumerate(fp.points):
        x = orc.fill_rng(F * pt.numel, qs.seed, pi, kind=1, lo=1.0, offset=qs.frame_offset * pt.numel)
        for _k in pt.consumers:
            up = orc.fill_rng(F * pt.numel, qs.seed + 500, ci, kind=1, lo=1.0,
                              offset=qs.frame_offset * pt.numel)
            ls = p[off:off + pt.channels]
            _, _, dls = orc.fq_backward(x, up, ls, F, pt.channels, pt.inner, want_dx=False)
            g.append(dls)
            off += pt.channels
            ci += 1
    g = np.concatenate(g + [np.zeros(qs.n_params - qs.n_act)])
    assert orc.adam(p, m, v, g, 0.9, 0.999, qs.lr, 1e-8, t) == 0
    return g


def test_qat_step_matches_oracle_over_steps(qfb, orc, cuda):
    import torch
    from paper_2511_12653_b200.frontend import QatStep
    F = 3
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    qs = QatStep(ctx, frames=F, seed=9, device=cuda, h=32, w=64)
    p = qs.params.cpu().numpy().copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for t in (1, 2, 3):
        with torch.cuda.stream(stream):
            qs.run()
        ctx.sync()
        if t == 1:
            # distillation: loss values and gradients per frame and pair
            loss = qs.losses()
            for f in range(F):
                for k, (c, s, tt, d) in enumerate(qs.feat):
                    st, o2, ds = orc.distill_pair(s[f].cpu().numpy(), tt[f].cpu().numpy(), qs.lam, 1.0 / F)
                    assert st == 0
                    assert loss[f, k].cpu().numpy().tobytes() == o2.tobytes()
                    assert np.array_equal(d[f].cpu().numpy().view(np.uint32), ds.view(np.uint32))
        g = oracle_step(orc, qs, p, m, v, t)
        assert qs.grads.cpu().numpy().tobytes() == g.tobytes(), t
        assert qs.params.cpu().numpy().tobytes() == p.tobytes(), t
        assert qs.m.cpu().numpy().tobytes() == m.tobytes(), t
        assert qs.adam.counters.cpu().tolist() == [t, 0, 0]
    ctx.close()


def test_qat_step_graph_replays_are_successive_steps(qfb, cuda):
    """resolve='device' + the local fold: the whole step captured once; three
    replays equal three eager steps bitwise (the counter, the device
    resolve and Adam all advance), and stay within the documented ulp
    tolerance of the host-resolved (bitwise-reference) steps."""
    import torch
    from paper_2511_12653_b200.frontend import QatStep
    stream = torch.cuda.Stream(device=cuda)
    ctx = qfb.Context(0, stream.cuda_stream)
    kw = dict(frames=2, seed=4, device=cuda, h=32, w=64)
    # an eager step of a fourth instance sizes the context's scratch (growth
    # under capture is refused); capture itself executes nothing
    with torch.cuda.stream(stream):
        QatStep(ctx, resolve="device", **kw).run()
    ctx.sync()
    a = QatStep(ctx, resolve="device", **kw)
    b = QatStep(ctx, resolve="device", **kw)
    h = QatStep(ctx, resolve="host", **kw)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        a.run()
    ctx.sync()
    for _ in range(3):
        g.replay()
        with torch.cuda.stream(stream):
            b.run()
            h.run()
    stream.synchronize()
    ctx.sync()
    assert torch.equal(a.params, b.params) and torch.equal(a.grads, b.grads)
    assert a.adam.counters.cpu().tolist() == [3, 0, 0]
    assert torch.allclose(a.params, h.params, rtol=1e-9, atol=1e-15)
    ctx.close()


def test_nccl_rank_comm_exchange_single_rank(qfb, cuda):
    """qfb_nccl_get_unique_id + qfb_nccl_comm_init_rank (one process per
    GPU) on a one-rank communicator: the QAT step with the NCCL
    gather-fold equals the step with the local fold, bitwise."""
    import torch
    from paper_2511_12653_b200.frontend import NcclGatherFold, QatStep
    if not qfb.nccl_available():
        pytest.fail("libqfb found no NCCL library on a GPU box")
    ctx = qfb.default_context(0)
    uid = qfb.nccl_unique_id()
    comm = qfb.NcclRankComm(uid, 1, 0, 0)
    try:
        kw = dict(frames=3, seed=6, device=cuda, h=32, w=64)
        a = QatStep(ctx, **kw)
        ex = NcclGatherFold(ctx, comm, 3, a.n_act, device=cuda)
        b = QatStep(ctx, exchange=ex, **kw)
        a.run()
        b.run()
        ctx.sync()
        assert torch.equal(a.grads, b.grads) and torch.equal(a.params, b.params)
    finally:
        comm.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
import paper_2511_12653_b200 as q
from paper_2511_12653_b200.frontend import QatStep, GlooGatherFold
dist.init_process_group("gloo")
r, ws = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
ctx = q.Context(0)
F = 4 // ws
qs = QatStep(ctx, frames=F, seed=8, device=dev, h=32, w=64, frame_offset=r * F, total_frames=4,
             exchange=GlooGatherFold(ctx) if ws > 1 else None)
for _ in range(2):
    qs.run()
ctx.sync()
np.save(os.path.join({out!r}, f"params_{{ws}}_{{r}}.npy"), qs.params.cpu().numpy())
np.save(os.path.join({out!r}, f"grads_{{ws}}_{{r}}.npy"), qs.grads.cpu().numpy())
dist.barrier()
dist.destroy_process_group()
"""


def test_two_rank_step_replicas_equal_single_rank(tmp_path):
    """Frames sharded over two ranks, exchange before Adam: after two steps
    both replicas hold the same bits, equal to one rank holding all four
    frames."""
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT, out=str(tmp_path)))
    for n in (1, 2):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
    one = np.load(tmp_path / "params_1_0.npy")
    for k in (0, 1):
        assert np.load(tmp_path / f"params_2_{k}.npy").tobytes() == one.tobytes(), k
        assert np.load(tmp_path / f"grads_2_{k}.npy").tobytes() == np.load(tmp_path / "grads_1_0.npy").tobytes()
