import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import test_gpu_multirank as T
from oracle import oracle as O
from paper_2604_25728_b200 import sqngd, configs as CF
for eng in ("fft", "cheb"):
    c = T.CASES[0].with_(loss_mode=CF.LOSS_LSE, beta_or_p=60.0, doppler_engine=T.ENGINES[eng])
    z, rho, q, w = T.inputs_for(c, 91)
    res = T.on_ranks(c, 2, lambda ctx, r: T.eval_all(ctx, z, rho, w))
    single = T.eval_all(sqngd.Context(c), z, rho, w)
    refB, _, _ = O.loss_grad(c, q["s_soft"], w, want_w=False)
    refA, _, _ = O.loss_grad(c, q["s_hard"], w, want_s=False)
    for key, ref in (("mA", refA), ("mB", refB)):
        for r in range(c.R):
            print(eng, key, r, "sharded", [round(res[0][key][r][k], 9) for k in ("loss_wpsl", "loss_snrl", "wpsl")],
                  "single", [round(single[key][r][k], 9) for k in ("loss_wpsl", "loss_snrl", "wpsl")],
                  "oracle", [round(ref[r][k], 9) for k in ("loss_wpsl", "loss_snrl", "wpsl")])
    for k in ("gw", "gz", "gr"):
        print(eng, k, np.linalg.norm(res[0][k] - single[k]) / np.linalg.norm(single[k]))
