"""Where the end-to-end (host-buffer) step time goes at C3: the bench's e2e loop with the host->device
copy, the device->host copies, both or neither inside the events (state and outputs in one flat
allocation each, as in bench.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402

c = CF.C3
dev = torch.device("cuda")
side = torch.cuda.Stream()
torch.cuda.set_stream(side)
ctx = sqngd.Context(c)
z = torch.as_tensor(inputs.phase_params(1, c.M, c.N, c.index), device=dev)
rho = torch.as_tensor(inputs.init_thresholds(1, c.B, c.r_n), device=dev)
w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
st = ctx.new_state(z, rho, w)
keys = ["z", "rho", "w", "m_z", "v_z", "m_rho", "v_rho", "m_w", "v_w"]
sizes = {k: st[k].numel() * (2 if st[k].is_complex() else 1) for k in keys}
flat = torch.empty(sum(sizes.values()), dtype=torch.float32, device=dev)
est, o = {"t_a": 0, "t_b": 0}, 0
for k in keys:
    v = flat[o:o + sizes[k]]
    v = v.view(torch.complex64) if st[k].is_complex() else v
    est[k] = v.view(st[k].shape)
    est[k].copy_(st[k])
    o += sizes[k]
hist = torch.zeros((1, 20), dtype=torch.float64, device=dev)
hard = torch.empty(sqngd.METRICS_BYTES, dtype=torch.uint8, device=dev)
host_state = flat.cpu().pin_memory()
host_hist = torch.empty_like(hist, device="cpu").pin_memory()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.current_stream()
for mode in ("step", "step", "step", "step", "both", "step", "both", "step"):
    for i in range(3):
        ctx.step(est, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(10):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if mode in ("h2d", "both"):
            flat.copy_(host_state, non_blocking=True)
        ctx.step(est, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
        if mode in ("d2h", "both"):
            host_state.copy_(flat, non_blocking=True)
            host_hist.copy_(hist, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    print(f"{mode:5s}: {tot / 10 * 1e3:8.1f} us per step", flush=True)
