"""The backward's HBM traffic pattern (read x and upstream, write d_input,
12 B/elem f32 over the 22 DPVO quant points of one frame) driven through
the forward chain kernel (a = x, b = up, one output): the memory ceiling of
this access pattern independent of the backward's tile structure."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200 import CChainDesc, check, lib  # noqa: E402
from paper_2511_12653_b200.frontend import FrontendQuantPass  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
ctx = q.Context(0, stream.cuda_stream)
fp = FrontendQuantPass(ctx, frames=1, dtype="f32", sets=2, seed=3, device=dev)
tables = []
for si in range(2):
    descs = []
    ci = 0
    for pi, p in enumerate(fp.points):
        for k in range(len(p.consumers)):
            d = CChainDesc()
            d.a = fp.sets[si]["x"][pi].data_ptr()
            d.b = fp.sets[si]["up"][ci].data_ptr()
            d.preact = 0
            d.y[0] = fp.dx[ci].data_ptr()
            d.scale[0] = fp.s32[ci].data_ptr()
            d.outer, d.channels, d.inner = 1, p.channels, p.inner
            d.n_out, d.act, d.dtype, d.q_max, d.flags = 1, 0, 0, 127, 0
            descs.append(d)
            ci += 1
    tables.append(((CChainDesc * len(descs))(*descs), len(descs)))
k = [0]


def run():
    t, n = tables[k[0] % 2]
    k[0] += 1
    check(lib().qfb_fq_chain_multi(ctx.handle, t, n))


for _ in range(5):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(200):
    run()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 200
bytes_ = fp.bytes_per_step()["bwd"]
print(json.dumps({"us": ms * 1e3, "gbps": bytes_ / (ms / 1e3) / 1e9, "bytes": bytes_}))
