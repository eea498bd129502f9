"""Driver for the ncu captures of the non-headline kernels (diagnostic tool):
config 3's quant->act->quant chain kernel (ReLU and GELU windows), config
5's int8 emission, and config 4's distillation + Adam kernels. Each workload
runs twice (warm-up, then the captured launch); run under

  ncu --set full -k regex:"ew_tma_kernel|leaf_sums|halve|cosine|adam" ...
      python tools/ncu_secondary.py [f32|f16]

and select launches with -s/-c (see tools/gpu_r02_u.sh)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_12653_b200 as q  # noqa: E402
from paper_2511_12653_b200.frontend import FrontendQuantPass, QatStep, WindowChainPass  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "f32"
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["relu", "gelu", "int8", "qat"]
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
ctx = q.Context(0, stream.cuda_stream)
for w in which:
    if w in ("relu", "gelu"):
        wp = WindowChainPass(ctx, frames=15, patches=96, gelu=(w == "gelu"), dtype=dt, device=dev)
        for _ in range(2):
            wp.run()
        ctx.sync()
        print(w, "bytes per window", wp.bytes_per_run(), flush=True)
        del wp
    elif w == "int8":
        fp = FrontendQuantPass(ctx, frames=8, dtype=dt, sets=1, seed=11, device=dev, int8_out=True)
        for _ in range(2):
            fp.forward(0)
        ctx.sync()
        print("int8 bytes per launch", fp.bytes_per_step()["fwd_int8"], flush=True)
        del fp
    elif w == "qat":
        st = QatStep(ctx, frames=8, dtype=dt, device=dev)
        for _ in range(2):
            st.run()
        ctx.sync()
        print("qat bytes per step", st.bytes_per_step(), flush=True)
        del st
    torch.cuda.empty_cache()
