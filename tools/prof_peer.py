"""Launch durations of the peer-memory combine kernels at 1 rank (their own window): C3 and C5 payloads.
  ncu --metrics gpu__time_duration.sum -k regex:"k_world|k_peer" python tools/prof_peer.py C5
SQNGD_PEER_FUSED=0 selects pack + k_peer_allreduce + unpack instead of k_world_peer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2604_25728_b200 import configs as CF
from paper_2604_25728_b200 import inputs, sqngd

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
c = CF.CONFIGS[name].with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0)
ctx = sqngd.Context(c, nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)
ctx.enable_peer_allreduce()
z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N) for r in range(c.R)])
rho = inputs.init_thresholds(c.R, c.B, c.r_n)
zt, rt = torch.as_tensor(z, device="cuda"), torch.as_tensor(rho, device="cuda")
w = ctx.quantize(zt, rt, soft=False, want_b=False, want_dq=False)["s_hard"]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(4):
    if i == 1:
        ev[0].record()
    met, gz, gr = ctx.af_loss_grad(zt, rt, w, sqngd.WRT_TRANSMIT)
ev[1].record()
ctx.sync()
print(name, "Step-B loss+grad evaluation (peer backend, 1 rank):", ev[0].elapsed_time(ev[1]) / 3, "ms; loss", ctx.metrics(met)[0]["loss"])
