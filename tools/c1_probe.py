"""Config-1 per-tensor forward ([1,128,120,160], 128 rotating maps) as a
CUDA graph of 128 calls: us per call. Usage: python tools/c1_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_12653_b200 as q  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(st)
ctx = q.Context(0, st.cuda_stream)
n = 128 * 120 * 160
L = q.lib()
xs = torch.empty((128, n), device=dev)
q.check(L.qfb_fill_rng(ctx.handle, 0, xs.data_ptr(), xs.numel(), 1, 0, 0, 1, 1.0, 0.0))
ys = torch.empty_like(xs)
s = torch.tensor([0.0315], dtype=torch.float32, device=dev)
k = [0]


def one():
    i = k[0] % 128
    k[0] += 1
    q.check(L.qfb_fq_fwd(ctx.handle, 0, xs[i].data_ptr(), ys[i].data_ptr(), 1, 1, n, s.data_ptr(), 127, 0))


for _ in range(8):
    one()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(128):
        one()
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(5):
    g.replay()
e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (5 * 128)
print(json.dumps({"us_per_call": us, "gbps": 2 * n * 4 / us / 1e3,
                  "env": {k2: os.environ.get(k2) for k2 in ("QFB_DISABLE_TMA_FWD", "QFB_FWD_STAGES", "QFB_PDL")}}))
