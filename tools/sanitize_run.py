"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): C1 and a ragged case on both
engines -- forward with the map, Step-A / Step-B loss+grad (LSE, p-norm, MAX), one sqngd_step through the
CUDA graph, the generator, and a 2-rank loopback evaluation.  python tools/sanitize_run.py"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF, inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402


def T(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def run(c):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=3)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    ctx = sqngd.Context(c)
    q = ctx.quantize(T(z), T(rho))
    w = q["s_hard"].clone()
    ctx.af_forward(q["s_hard"], w, want_map=True)
    ctx.af_loss_grad(T(z), T(rho), w, sqngd.WRT_FILTERS)
    ctx.af_loss_grad(T(z), T(rho), w, sqngd.WRT_TRANSMIT)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st = ctx.new_state(T(z), T(rho), w)
        hard = torch.empty(c.R * sqngd.METRICS_BYTES, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            ctx.step(st, sqngd.BLOCK_AB, hard_met=hard)
    torch.cuda.synchronize()
    ctx.sync()
    ctx.close()


for eng in (sqngd.ENGINE_FFT, sqngd.ENGINE_CHEBYSHEV):
    for mode, bp in ((CF.LOSS_LSE, 200.0), (CF.LOSS_PNORM, 16.0), (CF.LOSS_MAX, 0.0)):
        run(CF.C1.with_(loss_mode=mode, beta_or_p=bp, doppler_engine=eng, n_h=2, n_x=2))
    run(Cfg("rag", M=3, N=37, B=8, K=21, f_lo=-0.5, f_hi=0.5, R=2, r_n=3, n_h=2, n_x=2, doppler_engine=eng))
# generator mode
cg = CF.C1.with_(net_width=32, net_depth=2, n_h=1, n_x=2)
ctx = sqngd.Context(cg)
th = T(inputs.net_params(1, cg.M * cg.N, 32, 2, config_index=1))
y0 = T(inputs.net_input(1, cg.M, cg.N, cg.B, config_index=1))
zg = ctx.net_forward(th, y0)
rho = T(inputs.init_thresholds(1, cg.B, cg.r_n))
w = ctx.quantize(zg, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
st = ctx.new_state(zg, rho, w, theta=th, y0=y0)
ctx.step(st, sqngd.BLOCK_AB)
ctx.sync()
ctx.close()
# 2-rank loopback
c = CF.C1.with_(R=2, doppler_engine=sqngd.ENGINE_CHEBYSHEV)
lb = sqngd.Loopback(2)
ctxs = [sqngd.Context(c, loopback=lb, rank=r) for r in range(2)]
z = inputs.phase_params(c.R, c.M, c.N, config_index=3)
rho = inputs.init_thresholds(c.R, c.B, c.r_n)


def work(r):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        q = ctxs[r].quantize(T(z), T(rho))
        ctxs[r].af_loss_grad(T(z), T(rho), q["s_hard"], sqngd.WRT_TRANSMIT)
        s.synchronize()
        ctxs[r].sync()


th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
for x in ctxs:
    x.close()
lb.close()
print("sanitize workload ok")
