"""sqngd_step(A+B) replayed a few times at a BASELINE config (for launch lists / ncu).
python tools/step_loop.py [C3] [steps] [engine: auto|fft|cheb] [net: 0|1 (ResNet generator 5 x 128)]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
eng = {"fft": 1, "cheb": 2}.get(sys.argv[3] if len(sys.argv) > 3 else "auto", 0)
net = len(sys.argv) > 4 and sys.argv[4] == "1"
c = CF.CONFIGS[name].with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0, doppler_engine=eng)
if net:
    c = c.with_(net_width=128, net_depth=5)
z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N) for r in range(c.R)])
rho = inputs.init_thresholds(c.R, c.B, c.r_n)
side = torch.cuda.Stream()
torch.cuda.set_stream(side)
ctx = sqngd.Context(c)
zt, rt = torch.as_tensor(z, device="cuda"), torch.as_tensor(rho, device="cuda")
kw = {}
if net:
    kw = dict(theta=torch.as_tensor(inputs.net_params(c.R, c.M * c.N, 128, 5, c.index), device="cuda"),
              y0=torch.as_tensor(inputs.net_input(c.R, c.M, c.N, c.B, c.index), device="cuda"))
    zt = ctx.net_forward(kw["theta"], kw["y0"])
st = ctx.new_state(zt, rt, ctx.quantize(zt, rt, soft=False, want_b=False, want_dq=False)["s_hard"], **kw)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(steps + 2):
    if i == 2:
        ev[0].record()
    ctx.step(st, sqngd.BLOCK_AB)
ev[1].record()
torch.cuda.synchronize()
ctx.sync()
print(f"{name} engine={ctx.engine_info()['engine']}: {ev[0].elapsed_time(ev[1]) / steps:.3f} ms/step")
