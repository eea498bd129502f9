"""QFB_OPT_BWD_ASYNC_FINISH: the backward's finisher on the context's side
stream. After a join point (qfb_ctx_join, the next backward call, or
qfb_ctx_sync) the scale gradients are bit-identical to the stream-ordered
finisher's, eagerly and inside a captured CUDA graph (which must join before
the capture ends); the option validates its value and turning it off
joins."""
import pytest

pytestmark = pytest.mark.gpu


def grads(q, cuda, async_finish, graph, frames=1, steps=3):
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass
    stream = torch.cuda.Stream(device=cuda)
    ctx = q.Context(0, stream.cuda_stream)
    fp = FrontendQuantPass(ctx, frames=frames, dtype="f32", sets=2, seed=5, device=cuda, h=240, w=320)
    out = []
    with torch.cuda.stream(stream):
        fp.forward(0)
        fp.backward(0)  # eager: sizes the workspaces
        ctx.sync()
        if async_finish:
            ctx.set_option(q.OPT_BWD_ASYNC_FINISH, 1)
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for k in range(steps):
                    fp.forward(k % 2)
                    fp.backward(k % 2)
                ctx.join()
            g.replay()
        else:
            for k in range(steps):
                fp.forward(k % 2)
                fp.backward(k % 2)  # joins the previous finisher first
        ctx.join()
        out.append(fp.scale_grads().clone())
        dx = [t.clone() for t in fp.dx]
        if async_finish:
            ctx.set_option(q.OPT_BWD_ASYNC_FINISH, 0)
    ctx.sync()
    torch.cuda.synchronize(cuda)
    res = (out[0].cpu(), [t.cpu() for t in dx])
    ctx.close()
    return res


@pytest.mark.parametrize("graph", [False, True])
def test_async_finisher_matches_stream_order(qfb, cuda, graph):
    import torch
    g0, dx0 = grads(qfb, cuda, False, graph)
    g1, dx1 = grads(qfb, cuda, True, graph)
    assert torch.equal(g0.view(torch.int64), g1.view(torch.int64))
    for a, b in zip(dx0, dx1):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_async_finisher_option_validation(qfb, cuda):
    ctx = qfb.Context(0)
    with pytest.raises(qfb.ValueError):
        ctx.set_option(qfb.OPT_BWD_ASYNC_FINISH, 2)
    ctx.set_option(qfb.OPT_BWD_ASYNC_FINISH, 1)
    ctx.join()  # nothing pending: a no-op
    ctx.set_option(qfb.OPT_BWD_ASYNC_FINISH, 0)
    ctx.close()
