"""Profiling driver: C3 (or argv[1]) forward and Step-B loss+grad through the C-ABI, a few calls each
(for ncu -k regex:k_lrt).  python tools/prof_lr.py [C3] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF, inputs, sqngd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
want_map = len(sys.argv) > 3 and sys.argv[3] == "map"  # forward with the |A| map written
c = CF.CONFIGS[name].with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0)
z = torch.as_tensor(np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N)
                              for r in range(c.R)]), device="cuda")
rho = torch.as_tensor(inputs.init_thresholds(c.R, c.B, c.r_n), device="cuda")
ctx = sqngd.Context(c)
w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
for _ in range(reps):
    ctx.af_forward(w, w, want_map=want_map)
    ctx.af_loss_grad(z, rho, w, sqngd.WRT_TRANSMIT)
torch.cuda.synchronize()
ctx.sync()
print("ok", ctx.engine_info())
