import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2511_12653_b200 as q
from paper_2511_12653_b200 import _lib, _vp, check
dev = torch.device('cuda:0'); st = torch.cuda.Stream(device=dev); torch.cuda.set_stream(st)
ctx = q.Context(0, st.cuda_stream)
F = 64
feat = []
for c in (128, 384):
    s = torch.randn((F, c, 120, 160), device=dev); t = torch.randn_like(s); d = torch.empty_like(s)
    out = torch.empty((F, 2), dtype=torch.float64, device=dev)
    feat.append((c, s, t, d, out))
for _ in range(3):
    for c, s, t, d, out in feat:
        check(_lib.qfb_distill_batch(ctx.handle, _vp(s.data_ptr()), _vp(t.data_ptr()), F, c, 19200, 1.0, 1/64, _vp(d.data_ptr()), _vp(out.data_ptr())))
torch.cuda.synchronize()
