"""Forward-only throughput of FrontendQuantPass at F frames per launch
(BASELINE config 5 uses 8): ms per launch and HBM fraction, CUDA events.
Usage: python tools/c5_probe.py [frames] [f32|f16] [int8]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200.frontend import FrontendQuantPass  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dt = sys.argv[2] if len(sys.argv) > 2 else "f32"
int8 = len(sys.argv) > 3 and sys.argv[3] == "int8"
dev = torch.device("cuda:0")
st = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(st)
ctx = q.Context(0, st.cuda_stream)
fp = FrontendQuantPass(ctx, frames=F, dtype=dt, sets=2, seed=11, device=dev, int8_out=int8)
for i in range(4):
    fp.forward(i % 2)
torch.cuda.synchronize()
R = int(os.environ.get("C5_REPS", "40"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(R):
    fp.forward(i % 2)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
b = fp.bytes_per_step()["fwd"]
if int8:  # input read once + 1 byte per quant-point element
    esz = 4 if dt == "f32" else 2
    b = sum(p.numel * F * esz + p.numel * F * len(p.consumers) for p in fp.points)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6551.0
print(json.dumps({"frames": F, "dtype": dt, "ms": ms, "frames_per_s": F / ms * 1e3, "gbps": b / ms / 1e6,
                  "frac": b / ms / 1e6 / peak, "int8": int8, "reps": R, "stages_env": os.environ.get("QFB_FWD_STAGES")}))
