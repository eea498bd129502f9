"""Multi-process (world_size 2, gloo, CPU) test of the multi-GPU host logic:
frames shard across ranks, per-frame scale-gradient rows are all-gathered
and folded in frame order — bit-identical to the single-process sequential
accumulation (the reference trainer's `g += grad` over frames,
frontend.hpp:222-228), which is what the NCCL path does on B200s."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

F, C, HW = 6, 5, 333


def data():
    rng = np.random.default_rng(42)
    x = rng.normal(0, 1, (F, C, HW)).astype(np.float32)
    up = rng.normal(0, 1, (F, C, HW)).astype(np.float32)
    ls = rng.uniform(-6, -2, C)
    return x, up, ls


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, ws, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle
    from paper_2511_12653_b200.dist import gather_fold, shard_frames
    orc = oracle.Oracle()
    x, up, ls = data()
    lo, hi = shard_frames(F, ws, rank)
    rows = []
    for f in range(lo, hi):
        _, _, g = orc.fq_backward(x[f], up[f], ls, 1, C, HW, want_dx=False)
        rows.append(g)
    total = gather_fold(torch.tensor(np.stack(rows)))
    q.put((rank, total.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_fold_is_bit_identical(orc):
    x, up, ls = data()
    _, _, want = orc.fq_backward(x, up, ls, F, C, HW, want_dx=False)   # outer = F, frame order
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == want.tobytes()


def test_shard_frames_covers_all():
    from paper_2511_12653_b200.dist import shard_frames
    for n in (1, 7, 64):
        for ws in (1, 2, 4, 8):
            spans = [shard_frames(n, ws, r) for r in range(ws)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(ws - 1))
