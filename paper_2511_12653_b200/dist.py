"""Multi-GPU plumbing for the scale-only QAT step.

Frames shard across ranks (one process per GPU); the only exchange is the
per-channel scale-gradient vector (fp64, ~7 KB per frame for the 902 DPVO
activation scales). To keep the result BIT-IDENTICAL at any GPU count —
equal to the single-process trainer's frame-order accumulation
(distill.hpp:227-250 -> frontend.hpp:222-228, `g += grad` per frame) — each
rank contributes its per-frame rows, the rows are all-gathered (NCCL on
GPUs, gloo in the CPU tests) and folded in global frame order. An
all-reduce would make the bits depend on the rank count and NCCL's
reduction order.
"""
from __future__ import annotations

from typing import Optional


def fold_rows(rows, into=None):
    """((into + r0) + r1) + ...  (or r0 + r1 + ... when into is None), in
    row order, elementwise IEEE double adds. A [R, n] float64 CUDA tensor is
    folded by one qfb_fold_rows launch; CPU tensors (gloo tests) by torch."""
    import torch
    if isinstance(rows, torch.Tensor) and rows.is_cuda and rows.dtype == torch.float64:
        from . import fold_rows_device
        return fold_rows_device(rows.reshape(rows.shape[0], -1), into).reshape(rows.shape[1:])
    rows = list(rows)
    acc = rows[0].clone() if into is None else into + rows[0]
    for r in rows[1:]:
        acc = acc + r
    return acc


def gather_fold(local_rows, group=None, into: Optional[object] = None):
    """All-gather each rank's [F_local, n] per-frame gradient rows (rank r
    holds global frames [r*F_local, (r+1)*F_local)) and fold them in global
    frame order. Returns the [n] total on every rank."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return fold_rows(local_rows, into)
    ws = dist.get_world_size(group)
    local_rows = local_rows.contiguous()
    out = torch.empty((ws * local_rows.shape[0],) + tuple(local_rows.shape[1:]),
                      dtype=local_rows.dtype, device=local_rows.device)
    dist.all_gather_into_tensor(out, local_rows, group=group)
    return fold_rows(out, into)


def shard_frames(n_frames: int, world_size: int, rank: int):
    """Contiguous frame shard of this rank (weak scaling when n_frames is a
    per-rank count times world_size)."""
    per = n_frames // world_size
    extra = n_frames % world_size
    lo = rank * per + min(rank, extra)
    hi = lo + per + (1 if rank < extra else 0)
    return lo, hi
