"""Fixed vs per-frame cost of the fused forward and backward launches:
time one launch over F frames for F = 1, 2, 4, 8, 16 (inputs rotated over
two sets) and fit t = a + b*F."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200.frontend import FrontendQuantPass  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(st)
ctx = q.Context(0, st.cuda_stream)
res = {}
for F in (1, 2, 4, 8, 16):
    fp = FrontendQuantPass(ctx, frames=F, sets=2, device=dev)
    out = {}
    for name, fn in (("fwd", fp.forward), ("bwd", fp.backward)):
        for i in range(4):
            fn(i % 2)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(10, 200 // F)
        a.record(st)
        for i in range(reps):
            fn(i % 2)
        b.record(st)
        torch.cuda.synchronize()
        out[name] = a.elapsed_time(b) / reps * 1e3
    res[F] = out
    del fp
    torch.cuda.empty_cache()
fit = {}
for name in ("fwd", "bwd"):
    Fs = np.array(list(res.keys()), dtype=float)
    ts = np.array([res[f][name] for f in res])
    b, a = np.polyfit(Fs, ts, 1)
    fit[name] = {"fixed_us": a, "per_frame_us": b}
print(json.dumps({"us": res, "fit": fit}))
