"""Device time of qfb_distill_batch for BASELINE config 4's distillation
(64 frames; fnet 128 and inet 384 channels at 120x160), CUDA events on the
context stream. Prints one JSON line (ms per call per pair type, GB/s of
the algorithmic bytes: read s, t once, write d_s)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200 import _lib, _vp, check  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(st)
ctx = q.Context(0, st.cuda_stream)
F = int(os.environ.get("FRAMES", "64"))
res = {}
for c in (128, 384):
    s = torch.randn((F, c, 120, 160), device=dev)
    t = torch.randn_like(s)
    d = torch.empty_like(s)
    out = torch.empty((F, 2), dtype=torch.float64, device=dev)

    def call():
        check(_lib.qfb_distill_batch(ctx.handle, _vp(s.data_ptr()), _vp(t.data_ptr()), F, c, 19200, 1.0,
                                     1.0 / F, _vp(d.data_ptr()), _vp(out.data_ptr())))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 10
    e0.record(st)
    for _ in range(R):
        call()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    res[f"c{c}_ms"] = ms
    res[f"c{c}_gbps"] = 3 * s.numel() * 4 / (ms / 1e3) / 1e9
    res[f"c{c}_out_checksum"] = float(out.sum().item()) + float(d.double().sum().item())
print(json.dumps(res))
