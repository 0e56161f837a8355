"""PSL-vs-iteration trajectory of the Alg. 1 driver on one GPU.

python tools/run_trajectory.py [C2] [T] [patience] [net: 0|1] [engine: auto|fft|cheb]

Runs sqngd_run (Alg. 1 outer iterations with the stopping rule) from the seeded start of the
config and prints one JSON line: the hard-waveform PSLR (dB, Eq. 48 on the hard WPSL) after every
outer iteration, the best snapshot's, the iterations run and the wall time on the device.
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
patience = int(sys.argv[3]) if len(sys.argv) > 3 else 0
net = len(sys.argv) > 4 and sys.argv[4] == "1"
eng = {"fft": 1, "cheb": 2}.get(sys.argv[5] if len(sys.argv) > 5 else "auto", 0)
c = CF.CONFIGS[name].with_(R=1, loss_mode=CF.LOSS_LSE, beta_or_p=200.0, doppler_engine=eng)
if net:
    c = c.with_(net_width=128, net_depth=5, lr_theta=1e-5)
side = torch.cuda.Stream()
torch.cuda.set_stream(side)
ctx = sqngd.Context(c)
rho = torch.as_tensor(inputs.init_thresholds(1, c.B, c.r_n), device="cuda")
kw = {}
if net:
    kw = dict(theta=torch.as_tensor(inputs.net_params(1, c.M * c.N, 128, 5, c.index), device="cuda"),
              y0=torch.as_tensor(inputs.net_input(1, c.M, c.N, c.B, c.index), device="cuda"))
    z = ctx.net_forward(kw["theta"], kw["y0"])
else:
    z = torch.as_tensor(inputs.phase_params(1, c.M, c.N, c.index), device="cuda")
w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]  # matched start (Q3)
met, _, _ = ctx.af_forward(w, w)
start = ctx.metrics(met)[0]["wpsl"]
st = ctx.new_state(z, rho, w, **kw)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
best, bw, bi, hist, res = ctx.run(st, T=T, patience=patience)
b.record()
torch.cuda.synchronize()
h = hist.cpu().numpy()[: res["iterations"], 0]
db = lambda v: 20 * math.log10(max(float(v), 1e-30))  # noqa: E731
out = {"config": name, "generator": net, "engine": ctx.engine_info()["engine"], "T": T, "patience": patience,
       "iterations": res["iterations"], "stopped": res["stopped"], "device_s": a.elapsed_time(b) / 1e3,
       "start_pslr_db": db(start), "best_pslr_db": db(bw.cpu().numpy()[0]), "best_iter": int(bi.cpu().numpy()[0]),
       "pslr_db": [round(db(v), 3) for v in h]}
print(json.dumps(out))
