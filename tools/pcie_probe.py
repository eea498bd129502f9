"""PCIe ceiling for the e2e number: pinned H2D, D2H and both concurrently
(two streams = two copy engines), bytes of one DPVO frame (config 2)."""
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_12653_b200.frontend import dpvo_quant_points, frame_bytes  # noqa: E402

pts = dpvo_quant_points()
h2d = sum(p.numel * 4 for p in pts) + sum(p.numel * 4 * len(p.consumers) for p in pts)
d2h = sum(p.numel * 4 * 2 * len(p.consumers) for p in pts)
dev = torch.device("cuda:0")
hin = torch.empty(h2d // 4, dtype=torch.float32).pin_memory()
hout = torch.empty(d2h // 4, dtype=torch.float32).pin_memory()
din = torch.empty(h2d // 4, dtype=torch.float32, device=dev)
dout = torch.empty(d2h // 4, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d_only():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    s1.synchronize()


def d2h_only():
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


r = {"h2d_MB": h2d / 1e6, "d2h_MB": d2h / 1e6}
for name, fn in (("h2d", h2d_only), ("d2h", d2h_only), ("both", both)):
    ms = timed(fn)
    r[name + "_ms"] = ms
r["h2d_GBps"] = h2d / r["h2d_ms"] / 1e6
r["d2h_GBps"] = d2h / r["d2h_ms"] / 1e6
r["both_frames_per_s_ceiling"] = 1000.0 / r["both_ms"]
print(json.dumps(r))
