import sys, os, json, torch
sys.path.insert(0, '/root/repo')
import paper_2511_12653_b200 as q
from paper_2511_12653_b200 import _lib, _vp, check
from paper_2511_12653_b200.frontend import QatStep
dev = torch.device('cuda:0'); st = torch.cuda.Stream(device=dev); torch.cuda.set_stream(st)
ctx = q.Context(0, st.cuda_stream)
qs = QatStep(ctx, frames=64, device=dev)
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n): fn()
    b.record(st); torch.cuda.synchronize(); return a.elapsed_time(b) / n
def distill():
    for k, (c, s, tt, d) in enumerate(qs.feat):
        hw = s.shape[2] * s.shape[3]
        check(_lib.qfb_distill_batch(ctx.handle, _vp(s.data_ptr()), _vp(tt.data_ptr()), 64, c, hw, 1.0, 1/64, _vp(d.data_ptr()), _vp(qs.loss_flat[k].data_ptr())))
print(json.dumps({"fwd": t(lambda: qs.fp.forward(0)), "bwd": t(lambda: qs.fp.backward(0)), "distill": t(distill), "step": t(qs.run)}))
