"""Where the e2e time goes: qfb_quant_pass_host over one DPVO frame with
(a) everything, (b) forward only (no backward inputs/outputs), (c) backward
only, (d) no d_input output; ms per frame over 10 calls."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200.frontend import dpvo_quant_points  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
ctx = q.Context(0, stream.cuda_stream)
L = q.lib()
cfg = q.QuantConfig().to_c()
rng = np.random.default_rng(0)
pts = dpvo_quant_points()
keep = []
host = []
for p in pts:
    hx = torch.randn(p.numel).pin_memory()
    cons = []
    for _ in p.consumers:
        ls = np.log(np.expm1(np.exp(rng.uniform(np.log(1e-3), np.log(0.1), p.channels))))
        sc = np.array(q.resolve_scale(ls.tolist()), dtype=np.float64)
        hup = torch.randn(p.numel).pin_memory()
        hy = torch.empty(p.numel).pin_memory()
        hdx = torch.empty(p.numel).pin_memory()
        dls = np.zeros(p.channels)
        cons.append((ls, sc, hup, hy, hdx, dls))
        keep += [ls, sc, hup, hy, hdx, dls]
    keep.append(hx)
    host.append((p, hx, cons))


def table(fwd=True, bwd=True, dx=True):
    arr = []
    for p, hx, cons in host:
        hp = q.CHostPoint()
        hp.x = hx.data_ptr()
        hp.outer, hp.channels, hp.inner, hp.n_out = 1, p.channels, p.inner, len(cons)
        for k, (ls, sc, hup, hy, hdx, dls) in enumerate(cons):
            hp.s[k] = sc.ctypes.data
            hp.y[k] = hy.data_ptr() if fwd else None
            hp.log_s[k] = ls.ctypes.data if bwd else None
            hp.up[k] = hup.data_ptr() if bwd else None
            hp.dx[k] = hdx.data_ptr() if (bwd and dx) else None
            hp.d_log_s[k] = dls.ctypes.data if bwd else None
        arr.append(hp)
    return (q.CHostPoint * len(arr))(*arr), len(arr)


res = {}
for name, kw in [("all", {}), ("fwd_only", {"bwd": False}), ("bwd_only", {"fwd": False}),
                 ("no_dx", {"dx": False}), ("all_again", {})]:
    t, n = table(**kw)
    q.check(L.qfb_quant_pass_host(ctx.handle, 0, t, n, ctypes.byref(cfg)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        q.check(L.qfb_quant_pass_host(ctx.handle, 0, t, n, ctypes.byref(cfg)))
    torch.cuda.synchronize()
    res[name] = (time.perf_counter() - t0) * 100.0  # ms per call
print(json.dumps(res))
