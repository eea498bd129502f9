"""The device entry points are CUDA-graph capturable: descriptor tables
travel as kernel parameters, workspaces are sized on first use, the
backward finisher is stateless. A captured fwd+bwd step replays bit-exactly."""
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
