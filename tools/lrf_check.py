"""k_lrf (tcgen05 forward) against k_lrt (mma.sync forward) on the same inputs: maps and metrics.
python tools/lrf_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402


def one(c, seed, matched):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=seed)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    out = {}
    for flag in ("0", "1"):
        os.environ["SQNGD_LRF"] = flag
        ctx = sqngd.Context(c)
        zt, rt = torch.as_tensor(z, device="cuda"), torch.as_tensor(rho, device="cuda")
        s = ctx.quantize(zt, rt)["s_hard"]
        w = s.clone() if matched else s * torch.exp(0.3j * torch.cos(0.41 * torch.arange(c.N, device="cuda")))
        w = w.to(torch.complex64)
        res = []
        for _ in range(2):
            met, p, amap = ctx.af_forward(s, w, want_map=True)
            res.append((ctx.metrics(met), amap.clone()))
        ctx.sync()
        out[flag] = res
        ctx.close()
    os.environ.pop("SQNGD_LRF")
    (m0, a0), (m1, a1) = out["0"][0], out["1"][0]
    d = (a1 - a0).abs().max().item() / c.N
    print(f"{c.name} R={c.R} M={c.M} N={c.N} K={c.K} matched={matched}: map max|d|/N {d:.2e}  "
          f"loss {m0[0]['loss']:.6e} vs {m1[0]['loss']:.6e}  wpsl {m0[0]['wpsl']:.6e} vs {m1[0]['wpsl']:.6e}  "
          f"argmax {m0[0]['argmax_auto']} vs {m1[0]['argmax_auto']}  2nd call same: "
          f"{torch.equal(out['1'][0][1], out['1'][1][1])}")
    if d > 1e-5:
        diff = (a1 - a0).abs()
        idx = torch.nonzero(diff > 1e-3 * c.N)
        print("   bad cells:", idx.shape[0], idx[:8].tolist())


for c, matched in [(Cfg("c1", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5, r_n=4, doppler_engine=2), True),
                   (Cfg("c1", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5, r_n=4, doppler_engine=2), False),
                   (Cfg("rag", M=3, N=37, B=8, K=21, f_lo=-0.5, f_hi=0.5, R=2, r_n=3, doppler_engine=2), False),
                   (Cfg("c2", M=4, N=256, B=8, K=129, f_lo=-0.5, f_hi=0.5, r_n=4, doppler_engine=2), False),
                   (Cfg("c3s", M=2, N=1024, B=16, K=257, f_lo=-0.5, f_hi=0.5, r_n=4, doppler_engine=2), False)]:
    one(c, 3, matched)
