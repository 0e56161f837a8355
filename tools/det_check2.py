"""Determinism probe at kernel granularity (R = 2): repeated calls on identical inputs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402

c = Cfg("run", M=2, N=32, B=4, K=9, f_lo=-0.5, f_hi=0.5, r_n=4, R=2, n_h=1, n_x=1, lr_w=0.3, lr_z=3e-2,
        doppler_engine=1)
z = inputs.phase_params(c.R, c.M, c.N, config_index=31)
rho = inputs.random_sorted_thresholds(c.R, c.B, c.r_n, 5)
w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
z, rho, w = (torch.as_tensor(a, device="cuda") for a in (z, rho, w))
ctx = sqngd.Context(c)


def rep(name, fn, n=200):
    ref = [t.clone() for t in fn()]
    bad = 0
    for _ in range(n):
        out = fn()
        if not all(torch.equal(a, b) for a, b in zip(ref, out)):
            bad += 1
    print(f"{name}: {bad}/{n} differ", flush=True)


rep("quantize", lambda: [v for v in ctx.quantize(z, rho).values()])
rep("loss_grad_A", lambda: [ctx.af_loss_grad(z, rho, w, sqngd.WRT_FILTERS)[1].clone()])
rep("loss_grad_B", lambda: [t.clone() for t in ctx.af_loss_grad(z, rho, w, sqngd.WRT_TRANSMIT)[1:]])
for blk in (1, 2):
    def one_step():
        st = ctx.new_state(z, rho, w)
        ctx.step(st, blk)
        return [st[k] for k in ("z", "rho", "w", "m_z", "v_z", "m_rho", "v_rho")]
    rep(f"step block {blk}", one_step, 100)
