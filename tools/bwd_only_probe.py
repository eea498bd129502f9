"""The backward alone, launched back to back (no forward between): the
steady-state time of the backward kernel (+ finisher) on one frame of
BASELINE config 2, for comparison with tools/bwd_traffic_probe.py (the same
traffic through the forward chain kernel). QFB_BWD_VARIANT selects the
probes (8: memory pipeline only, 16: arithmetic only)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200.frontend import FrontendQuantPass  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "f32"
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
ctx = q.Context(0, stream.cuda_stream)
if os.environ.get("QFB_HALF_FP32") == "1":
    ctx.set_option(q.OPT_BWD_HALF_FP32, 1)
fp = FrontendQuantPass(ctx, frames=1, dtype=dt, sets=2, seed=3, device=dev)
for i in range(5):
    fp.backward(i % 2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for i in range(200):
    fp.backward(i % 2)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 200
b = fp.bytes_per_step()["bwd"]
# the main pass alone: the library records an event between the main pass
# and the finisher (QFB_OPT_MAIN_PASS_EVENT)
st_ev = [torch.cuda.Event(enable_timing=True) for _ in range(50)]
mid_ev = [torch.cuda.Event(enable_timing=True) for _ in range(50)]
for e in mid_ev:
    e.record(stream)
torch.cuda.synchronize()
for i in range(50):
    st_ev[i].record(stream)
    ctx.set_option(q.OPT_MAIN_PASS_EVENT, mid_ev[i].cuda_event)
    fp.backward(i % 2)
ctx.set_option(q.OPT_MAIN_PASS_EVENT, 0)
torch.cuda.synchronize()
main_ms = sum(a.elapsed_time(m) for a, m in zip(st_ev, mid_ev)) / 50
print(json.dumps({"dtype": dt, "variant": os.environ.get("QFB_BWD_VARIANT", "0"), "impl": os.environ.get("QFB_BWD_IMPL", "") + ("+h32" if os.environ.get("QFB_HALF_FP32") == "1" else ""), "us": ms * 1e3, "main_us": main_ms * 1e3, "main_frac": b / (main_ms / 1e3) / 1e9 / 6551.0,
                  "gbps": b / (ms / 1e3) / 1e9, "frac": b / (ms / 1e3) / 1e9 / 6551.0}))
