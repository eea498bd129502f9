"""The C-ABI scale-gradient exchange (qfb_nccl.cpp) on the one GPU of the
box: a single-device communicator from ncclCommInitAll. gather-fold must be
bit-identical to the row-order fold of the same rows (the single-GPU
trainer's frame order), all-reduce over one rank the identity. The
multi-rank host logic is covered with gloo in tests/test_dist_gloo.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gather_fold_single_rank(qfb, cuda):
    import torch
    if not qfb.nccl_available():
        pytest.fail("libqfb found no NCCL library on a GPU box")
    comms = qfb.NcclComms([0])
    try:
        rng = np.random.default_rng(3)
        rows = torch.from_numpy(rng.normal(0, 1, (5, 1494)) * 10.0 ** rng.integers(-8, 8, (5, 1494))).to(cuda)
        into = torch.from_numpy(rng.normal(0, 1, 1494)).to(cuda)
        got = qfb.gather_fold_scale_grads(comms[0], rows, 1, into=into)
        torch.cuda.synchronize()
        want = into.cpu().numpy().copy()
        for r in rows.cpu().numpy():
            want = want + r
        assert got.cpu().numpy().tobytes() == want.tobytes()
        g = rows[0].clone()
        qfb.allreduce_scale_grads(comms[0], g)
        torch.cuda.synchronize()
        assert torch.equal(g, rows[0])
    finally:
        comms.close()


def test_bad_arguments(qfb, cuda):
    ctx = qfb.default_context(0)
    with pytest.raises(qfb.ValueError):
        qfb.check(qfb.lib().qfb_gather_fold_scale_grads(ctx.handle, None, None, 1, 1, None, None, None))
