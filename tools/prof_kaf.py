"""Profiling driver: a few eager Step-A / Step-B loss+grad evaluations at a BASELINE config
(for ncu captures of the fused k_af kernels).  python tools/prof_kaf.py [C3] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = CF.CONFIGS[name].with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0,
                           doppler_engine={"fft": 1, "cheb": 2}.get(os.environ.get("SQNGD_ENGINE", ""), 0))
z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N) for r in range(c.R)])
rho = inputs.init_thresholds(c.R, c.B, c.r_n)
ctx = sqngd.Context(c)
zt, rt = torch.as_tensor(z, device="cuda"), torch.as_tensor(rho, device="cuda")
w = ctx.quantize(zt, rt)["s_hard"].clone()
for _ in range(reps):
    ctx.af_loss_grad(zt, rt, w, sqngd.WRT_FILTERS)
    ctx.af_loss_grad(zt, rt, w, sqngd.WRT_TRANSMIT)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
for _ in range(20):
    ctx.af_loss_grad(zt, rt, w, sqngd.WRT_FILTERS)
ev[1].record()
for _ in range(20):
    ctx.af_loss_grad(zt, rt, w, sqngd.WRT_TRANSMIT)
ev[2].record()
torch.cuda.synchronize()
print(f"{name}: af_loss_grad A {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.1f} us  B {ev[1].elapsed_time(ev[2]) / 20 * 1e3:.1f} us")
ctx.sync()
