"""Determinism probe: the same sqngd_step(A+B) sequence twice from the same start; reports the first
outer iteration at which any state tensor differs (R restarts, engine)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402

for R in (1, 2):
    for eng in (1, 2):
        for graph in (True, False):
            c = Cfg("run", M=2, N=32, B=4, K=9, f_lo=-0.5, f_hi=0.5, r_n=4, R=R, n_h=2, n_x=2, lr_w=0.3, lr_z=3e-2,
                    doppler_engine=eng)
            z = inputs.phase_params(c.R, c.M, c.N, config_index=31)
            rho = inputs.init_thresholds(c.R, c.B, c.r_n)
            w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
            z, rho, w = (torch.as_tensor(a, device="cuda") for a in (z, rho, w))
            ctx = sqngd.Context(c)
            stream = torch.cuda.Stream() if graph else torch.cuda.default_stream()
            hist = []
            with torch.cuda.stream(stream):
                for rep in range(2):
                    st = ctx.new_state(z, rho, w)
                    hard = torch.empty(c.R * sqngd.METRICS_BYTES, dtype=torch.uint8, device="cuda")
                    h = []
                    for t in range(16):
                        ctx.step(st, sqngd.BLOCK_AB, hard_met=hard)
                        h.append({k: st[k].clone() for k in ("z", "rho", "w", "m_w", "v_w")})
                    hist.append(h)
            torch.cuda.synchronize()
            first = None
            for t in range(16):
                for k in hist[0][t]:
                    if not torch.equal(hist[0][t][k], hist[1][t][k]):
                        d = (hist[0][t][k] - hist[1][t][k]).abs()
                        rr = [int(d[r].max() > 0) for r in range(R)]
                        first = (t + 1, k, rr, float(d.max()))
                        break
                if first:
                    break
            print(f"R={R} engine={eng} graph={graph}: first divergence {first}", flush=True)
            ctx.close()
