"""NEXT-3 reduced-T trend checks: the direction of PAPER.md Table II (larger
SNRL allowance mu -> lower APSL / CPSL) and Table III (wider Doppler range -> higher PSL) with
the Alg.-1 driver at C1 shape.  python tools/trend_table2.py [T] [R]"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF, inputs, sqngd  # noqa: E402


def best_psl(c, T, seed=7):
    ctx = sqngd.Context(c)
    z = torch.as_tensor(inputs.phase_params(c.R, c.M, c.N, config_index=seed), device="cuda")
    rho = torch.as_tensor(inputs.init_thresholds(c.R, c.B, c.r_n), device="cuda")
    w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
    st = ctx.new_state(z, rho, w)
    best, bw, bi, hist, res = ctx.run(st, T=T, patience=0, want_hist=False)
    q = ctx.quantize(best["z"], best["rho"], soft=False, want_b=False, want_dq=False)
    met, _, _ = ctx.af_forward(q["s_hard"], best["w"])
    m = ctx.metrics(met)
    ctx.sync()
    ctx.close()
    return [(r["apslr_db"], r["cpslr_db"], r["pslr_db"]) for r in m]


if __name__ == "__main__":
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    base = CF.C1.with_(R=R, loss_mode=CF.LOSS_LSE, beta_or_p=200.0)
    out = {"T": T, "R": R, "table2": {}, "table3": {}}
    for mu in (0.0, 0.5, 1.0, 1.5):
        v = np.array(best_psl(base.with_(mu_db=mu), T))
        out["table2"][mu] = {"apslr_db": v[:, 0].mean(), "cpslr_db": v[:, 1].mean(), "pslr_db": v[:, 2].mean()}
    for f in (0.1, 0.5, 3.0):
        v = np.array(best_psl(base.with_(f_lo=-f, f_hi=f), T))
        out["table3"][f] = {"apslr_db": v[:, 0].mean(), "cpslr_db": v[:, 1].mean(), "pslr_db": v[:, 2].mean()}
    print(json.dumps(out))
