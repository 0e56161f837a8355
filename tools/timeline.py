"""Device timeline of sqngd_step(A+B) replays (CUPTI kernel records through torch.profiler): per kernel
start / duration / gap to the previous kernel, grouped per evaluation, plus the per-kernel mean over the
profiled steps.  Unlike an ncu launch list this keeps the graph's concurrency and launch gaps.
python tools/timeline.py [C3] [steps] [engine: auto|fft|cheb] [out.json]"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = {"fft": 1, "cheb": 2}.get(sys.argv[3] if len(sys.argv) > 3 else "auto", 0)
out = sys.argv[4] if len(sys.argv) > 4 else None
e2e = len(sys.argv) > 5 and sys.argv[5] == "e2e"  # bench.py's e2e loop: state up, step, state + outputs down
c = CF.CONFIGS[name].with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0, doppler_engine=eng)
z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N) for r in range(c.R)])
rho = inputs.init_thresholds(c.R, c.B, c.r_n)
side = torch.cuda.Stream()
torch.cuda.set_stream(side)
ctx = sqngd.Context(c)
zt, rt = torch.as_tensor(z, device="cuda"), torch.as_tensor(rho, device="cuda")
st = ctx.new_state(zt, rt, ctx.quantize(zt, rt, soft=False, want_b=False, want_dq=False)["s_hard"])
hist = torch.zeros((c.R, c.n_h + c.n_x), dtype=torch.float64, device="cuda")
hard = torch.empty(c.R * sqngd.METRICS_BYTES, dtype=torch.uint8, device="cuda")
if e2e:
    keys = ["z", "rho", "w", "m_z", "v_z", "m_rho", "v_rho", "m_w", "v_w"]
    sizes = {k: st[k].numel() * (2 if st[k].is_complex() else 1) for k in keys}
    nst = sum(sizes.values())
    buf = torch.empty(4 * nst + hist.numel() * 8 + hard.numel(), dtype=torch.uint8, device="cuda")
    flat = buf[:4 * nst].view(torch.float32)
    est, o = {"t_a": st["t_a"], "t_b": st["t_b"]}, 0
    for k in keys:
        v = flat[o:o + sizes[k]]
        v = v.view(torch.complex64) if st[k].is_complex() else v
        est[k] = v.view(st[k].shape)
        est[k].copy_(st[k])
        o += sizes[k]
    hist = buf[4 * nst:4 * nst + hist.numel() * 8].view(torch.float64).view(hist.shape)
    hard = buf[4 * nst + hist.numel() * 8:]
    st = est
    host_buf = buf.cpu().pin_memory()


def one_step():
    if e2e:
        buf[:4 * nst].copy_(host_buf[:4 * nst], non_blocking=True)
    ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
    if e2e:
        host_buf.copy_(buf, non_blocking=True)


for _ in range(3):
    one_step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ev[0].record()
    for _ in range(steps):
        one_step()  # as bench.py times it
    ev[1].record()
    torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / steps
ks = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        nm = e.name
        if "memcpy" in nm.lower() or "memset" in nm.lower():
            print(f"non-kernel device activity: {nm} {e.time_range.elapsed_us():.2f} us at {e.time_range.start}")
            continue
        ks.append((e.time_range.start, e.time_range.end, nm.split("(")[0].replace("void ", "")[:48]))
ks.sort()
evals_per_step = c.n_h + c.n_x
# split into steps at k_set_t (the first kernel of every sqngd_step)
starts = [i for i, k in enumerate(ks) if "k_set_t" in k[2]]
rows = []
per = collections.defaultdict(list)
for si, s0 in enumerate(starts):
    s1 = starts[si + 1] if si + 1 < len(starts) else len(ks)
    seg = ks[s0:s1]
    t0 = seg[0][0]
    prev_end = t0
    for b, e, nm in seg:
        rows.append(dict(step=si, name=nm, start_us=b - t0, dur_us=e - b, gap_us=b - prev_end, abs_us=b - ks[0][0]))
        per[nm].append(e - b)
        prev_end = max(prev_end, e)
    if si == 0:
        print(f"step 0: {len(seg)} kernels, {(seg[-1][1] - t0):.1f} us device span")
print(f"{name}: {ms:.3f} ms/step (CUDA events, under the profiler), {evals_per_step} evals/step")
print(f"{'kernel':48s} {'n/step':>6s} {'mean us':>8s} {'sum/step us':>11s}")
nst = max(1, len(starts))
for nm, v in sorted(per.items(), key=lambda x: -sum(x[1])):
    print(f"{nm:48s} {len(v) / nst:6.1f} {np.mean(v):8.2f} {sum(v) / nst:11.1f}")
# one Step-A and one Step-B evaluation of step 1 in order (start, duration, gap)
s1 = [r for r in rows if r["step"] == min(1, nst - 1)]
print("\nstep 1 kernel order (start, dur, gap us):")
for r in s1[:60]:
    print(f"  {r['start_us']:8.1f} {r['dur_us']:7.2f} {r['gap_us']:6.2f}  {r['name']}")
gaps = [r["gap_us"] for r in rows if r["gap_us"] > 0]
for si in range(1, len(starts)):  # device idle between the end of step si-1 and the start of step si
    prev = [r for r in rows if r["step"] == si - 1]
    end = max(r["abs_us"] + r["dur_us"] for r in prev)
    first = min(r["abs_us"] for r in rows if r["step"] == si)
    print(f"idle before step {si}: {first - end:.1f} us")
print(f"\nidle between kernels: {sum(gaps) / nst:.1f} us/step over {len(gaps) / nst:.0f} gaps")
if out:
    json.dump(dict(config=name, ms_per_step=ms, rows=rows), open(out, "w"))
