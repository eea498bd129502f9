"""Frame pipelining probe: within a QAT chunk the scales are fixed
(distill.hpp:227-250), so the forward of frame k+1 does not depend on the
backward of frame k. Compare ms per frame of (a) the serial step graph
(fwd(k); bwd(k) on one stream) with (b) a two-stream graph of M frames where
bwd(k) runs on stream B after fwd(k) and fwd(k+1) proceeds on stream A.
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200.frontend import FrontendQuantPass  # noqa: E402


def main():
    dt = sys.argv[1] if len(sys.argv) > 1 else "f32"
    M = int(os.environ.get("M", "8"))
    R = int(os.environ.get("R", "100"))
    dev = torch.device("cuda", 0)
    sA = torch.cuda.Stream(device=dev)
    sB = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(sA)
    ctxA = q.Context(0, sA.cuda_stream)
    ctxB = q.Context(0, sB.cuda_stream)
    fp = FrontendQuantPass(ctxA, frames=1, dtype=dt, sets=2, seed=1, device=dev)
    for i in range(4):
        fp.forward(i % 2)
        fp.backward(i % 2)
        fp.backward(i % 2, ctx=ctxB)
    torch.cuda.synchronize()
    out = {}
    # (a) serial
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=sA):
        for k in range(M):
            fp.forward(k % 2)
            fp.backward(k % 2)
    # (b) pipelined
    g2 = torch.cuda.CUDAGraph()
    evs = [torch.cuda.Event() for _ in range(M)]
    with torch.cuda.graph(g2, stream=sA):
        for k in range(M):
            fp.forward(k % 2)
            evs[k].record(sA)
            sB.wait_event(evs[k])
            fp.backward(k % 2, ctx=ctxB)
        sA.wait_stream(sB)
    for name, g in (("serial", g1), ("pipelined", g2)):
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sA)
        for _ in range(R):
            g.replay()
        e1.record(sA)
        torch.cuda.synchronize()
        out[name + "_ms_per_frame"] = e0.elapsed_time(e1) / (R * M)
    # results identical: rerun the pipelined graph once more and compare grads
    g1.replay()
    torch.cuda.synchronize()
    a = fp.dls_flat.clone()
    g2.replay()
    torch.cuda.synchronize()
    out["grads_identical"] = bool(torch.equal(a, fp.dls_flat))
    out.update(dtype=dt, frames_per_graph=M, replays=R)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
