"""Benchmark of the SQNGD AF/CAF loss+gradient hot path (BASELINE.json metric).

A *step* is one Algorithm-1 outer iteration through the
public C-ABI call sqngd_step(block = A+B): n_h = 10 Step-A loss+gradient
evaluations (X_hard fixed, gradient to the filters, Adam, energy projection) and
n_x = 10 Step-B evaluations (soft quantizer, gradient to z and rho through Q_A,
Adam, threshold projection), with the hard-waveform metrics (loss, WAPSL / WCPSL /
WPSL, PSLR, SNRL) of the iterate the step starts from, scored by its first Step-A
evaluation -- every row of SURVEY.md §8(a).  value = loss+gradient evaluations per second over all ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

N > 1 (torchrun, one rank per GPU): every rank optimizes its own independent
seeded restart(s) (restart index = rank), no data-path collective -> "weak".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, parallel  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "loss+grad evals/s"


def fft_flops(P):
    return 5.0 * P * math.log2(P)


def work_model(c):
    """Algorithmic FP32 flops per launch of each fused kernel of the per-bin FFT engine
    (SURVEY.md §8(d)), per restart: 5 P log2 P per complex FFT, 6 per complex multiply, 7 / 10
    per cell.  The Doppler-modulated FFTs X = FFT(s e^{j2pi nf/N}) (K M of them) are done by
    k_xhat, not by the fused kernel, so they are not counted in its launch."""
    M, N, K, P = c.M, c.N, c.K, c.P
    cells = c.cells
    F = fft_flops(P)
    fwd_body = K * M * M * (6 * P + F) + 7 * cells      # slices: cross-spectrum + IFFT + cell epilogue
    F_A = 10 * cells + K * M * M * (F + 8 * P)
    F_B = 10 * cells + K * (M * M * (F + 8 * P) + M * (F + 6 * N))
    return {"fwd": fwd_body * c.R, "adjA": (fwd_body + F_A) * c.R, "adjB": (fwd_body + F_B) * c.R,
            "filter": M * F * c.R, "cells": cells * c.R}


def work_model_lr(c, Q):
    """Algorithmic work per launch of the Chebyshev engine's fused kernel k_lrt, split by
    the pipe that executes it (VERDICT r01 "What's weak" 2: only the cell epilogue runs on the FP32
    pipe; the Doppler contraction runs on the tensor pipe):
      fp32:   the cell epilogue of SURVEY.md §8(d): 7 flops per cell forward (|A|^2 3, sqrt 1, exp 1,
              sum 1, compare 1), 10 more with the gradient (cotangent);
      tensor: the Lagrange contraction At = sum_q l_q R_q and its adjoint in the symmetric form: per
              cell 2Q + 2 flops forward (Q/2 complex-by-real MACs for each of Pe, Po per bin pair,
              and the +/-), the same again for the adjoint."""
    cells = c.cells * c.R
    return {"fwd": {"fp32": 7 * cells, "tensor": (2 * Q + 2) * cells},
            "adjA": {"fp32": 17 * cells, "tensor": (4 * Q + 4) * cells},
            "adjB": {"fp32": 17 * cells, "tensor": (4 * Q + 4) * cells}, "cells": cells}


def tensor_peaks():
    """Dense tensor peaks per operand type (TFLOP/s): the measured bf16 burst figure of MEASURED_PEAKS.json
    times the nominal ratio of /opt/skills/guides/B200_PROFILING.md (FP16 = BF16: 1; TF32: 1.1 / 2.25)."""
    try:
        bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        src = "measured bf16 burst (MEASURED_PEAKS.json)"
    except Exception:
        bf16, src = 2250.0, "nominal bf16 (B200_PROFILING.md fallback)"
    return {"f16": bf16, "tf32": bf16 * 1.1 / 2.25, "basis": f"{src} x nominal dtype ratio (f16 1, tf32 1.1/2.25)"}


def traffic_bytes(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full
    capture (profiles/traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["dram_bytes_per_launch"]
        return d.get(kernel)
    except Exception:
        return None


def warp_instr(kernel, cfg_name):
    """Executed warp-instructions per launch of `kernel` at config `cfg_name` from the committed ncu
    capture (profiles/traffic.json), or None (a property of the kernel and the problem size)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["warp_instructions_per_launch"]
        return d.get(f"{kernel}@{cfg_name}")
    except Exception:
        return None


def issue_pipe(kernel, cfg_name, avg_ms, sms, sm_mhz):
    """Issue-slot use of the dominant kernel: its ncu-counted warp-instructions per launch over the live
    launch time, against one warp-instruction per clock per SM sub-partition (4 per SM)."""
    n = warp_instr(kernel, cfg_name)
    if not n:
        return None
    peak = sms * 4 * sm_mhz * 1e6
    ach = n / (avg_ms / 1e3)
    return {"achieved": ach / 1e9, "peak": peak / 1e9, "frac": ach / peak, "unit": "G warp-instr/s",
            "warp_instr_per_launch": n, "basis": f"ncu smsp__inst_executed.sum (profiles/traffic.json) / launch time; "
                                                 f"peak {sms} SM x 4 issue slots x {sm_mhz:.0f} MHz"}


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p.get("sm_max_mhz", 1965.0)), float(p.get("hbm_gbs", 6545.9)), "measured"
    except Exception:
        return 1965.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- oracle (CPU) leg
def oracle_sample(c, budget_s: float = 10.0):
    """One Step-B loss+gradient evaluation of the fp64 oracle (quantize -> AF -> loss ->
    adjoint sums -> chain to z, rho), measured on a sample of the workload's Doppler bins
    (evenly spaced, evaluated one bin at a time until `budget_s` is spent) and scaled to the
    full grid: the oracle's AF and adjoint cost is exactly linear in the bin count."""
    from oracle import oracle as O

    z = inputs.phase_params(1, c.M, c.N, c.index)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    order = np.linspace(0, c.K - 1, c.K).round().astype(int)
    order = np.concatenate([order[::max(1, c.K // 16)], order])      # spread the first picks
    t0 = time.perf_counter()
    q = O.quantize(c.with_(R=1), z, rho)
    t_q = time.perf_counter() - t0
    w = q["s_hard"]
    t_bins, nb, gs = 0.0, 0, None
    seen = set()
    for k in order:
        if k in seen:
            continue
        seen.add(k)
        f = c.f_lo + (c.f_hi - c.f_lo) * k / max(1, c.K - 1)
        cc = c.with_(R=1, K=1, f_lo=float(f), f_hi=float(f))
        t1 = time.perf_counter()
        _, _, gs = O.loss_grad(cc, q["s_soft"], w, want_w=False)
        t_bins += time.perf_counter() - t1
        nb += 1
        if t_bins >= budget_s:
            break
    t1 = time.perf_counter()
    O.chain(c.with_(R=1), z, rho, q["s_soft"], gs)
    t_chain = time.perf_counter() - t1
    return t_q + t_bins * c.K / nb + t_chain, nb


def cpu_info():
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count()
    return n


def run_reference(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_info()))
    times = []
    nb = 1
    t_wall = time.perf_counter()
    for i in range(args.warmup + args.steps):
        t, nb = oracle_sample(c, budget_s=2.0)
        if i >= args.warmup:
            times.append(t)
    t_wall = time.perf_counter() - t_wall
    per_eval = statistics.mean(times)
    v = 1.0 / per_eval
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_eval * 1e3 * 20, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "extrapolated": True,
        "extrapolation": f"each 'step' evaluates a bounded sample ({nb} of {c.K} Doppler bins of one Step-B loss+grad "
                         f"evaluation, ~2 s of CPU work) and scales the AF / adjoint time by K / {nb}; value and "
                         f"ms_per_step (20 evaluations per Alg. 1 outer iteration) are that extrapolation, not "
                         f"elapsed time: the whole run took {t_wall:.1f} s of wall clock",
        "sample_wall_s": t_wall,
        "config": config_dict(c),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "oracle",
                         "sample": f"Step-B loss+grad (quantize, AF, LSE loss, adjoint, chain) of the fp64 oracle with "
                                   f"{nb} of {c.K} Doppler bins evaluated, AF/adjoint time scaled by K/{nb}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(c):
    return {"workload": f"{c.name}: M={c.M} N={c.N} L={c.B} K={c.K} f=[{c.f_lo},{c.f_hi}] R={c.R}",
            "M": c.M, "N": c.N, "B": c.B, "K": c.K, "R_per_gpu": c.R, "P": c.P,
            "cells_per_eval": c.cells, "loss": {0: "max", 1: f"lse beta={c.beta_or_p}",
                                                  2: f"pnorm p={c.beta_or_p}"}[c.loss_mode],
            "step": "1 Alg.1 outer iteration: 10 Step-A + 10 Step-B loss+grad evals, Adam, projections, "
                    "hard-waveform metrics of the entry iterate (from the first Step-A evaluation)",
            "l2": "256 MiB L2 flush between timed steps (outside the per-step events)"}


# --------------------------------------------------------------------------- GPU leg
def work_sharded(args, world, rank, local, dev, stream, flush, name="C5"):
    """BASELINE.json's C5 (M=16, N=4096, K=513, 8 restarts) as ONE problem over the N ranks: the library's
    world > 1 mode (Chebyshev engine: each rank evaluates a slice of the R M (restart, transmit channel)
    rows; one grouped NCCL all-reduce per loss+grad evaluation, captured in the step's CUDA graph).
    value = loss+grad evals/s of the whole job (8 restarts x 20 per step / max-over-ranks step time)."""
    import torch

    from paper_2604_25728_b200 import sqngd

    c = CF.CONFIGS[name].with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0)
    def fresh_uid():  # one ncclUniqueId per communicator, rank 0's, broadcast
        if world == 1:
            return None
        import torch.distributed as dist

        obj = [sqngd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    uid = fresh_uid()
    z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N)
                  for r in range(c.R)])
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    steps, warm = max(2, min(args.steps, 5)), max(3, min(args.warmup, 3))

    def run(uid_, peer=False):
        ctx = sqngd.Context(c, device=local, nccl_uid=uid_, rank=rank, world=world)
        if peer:  # the library's own in-kernel all-reduce over peer memory instead of NCCL
            ctx.enable_peer_allreduce(rank, world)
        zt, rt = torch.as_tensor(z, device=dev), torch.as_tensor(rho, device=dev)
        w = ctx.quantize(zt, rt, soft=False, want_b=False, want_dq=False)["s_hard"]
        st = ctx.new_state(zt, rt, w)
        for _ in range(warm):
            ctx.step(st, sqngd.BLOCK_AB)
        ctx.sync()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(steps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            ctx.step(st, sqngd.BLOCK_AB)
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        ctx.sync()
        ms_ = parallel.max_over_ranks(sum(a.elapsed_time(b) for a, b in evs)) / steps
        info_ = ctx.engine_info()
        ctx.close()
        return ms_, info_

    ms, info = run(uid)
    # at N = 1, the same problem through the collective path over a 1-rank NCCL communicator (pack,
    # grouped NCCL all-reduce captured in the graph, unpack): the sharded code's own single-GPU cost
    ms_1r = run(sqngd.nccl_unique_id())[0] if world == 1 else None
    evals = (c.n_h + c.n_x) * c.R
    extra = {} if ms_1r is None else {"collective_path_1rank": {
        "value": evals / (ms_1r / 1e3), "ms_per_step": ms_1r,
        "what": "the same steps with an ncclUniqueId at world = 1: the sharded path and its grouped NCCL "
                "all-reduce over a 1-rank communicator"}}
    # the same sharded steps with the collective as ONE kernel of the library over peer memory
    # (sqngd_peer_export / sqngd_peer_attach; NEXT-4).  Between ranks it has never run (one GPU per box
    # here): a failure is reported, the NCCL numbers above stand.
    try:
        ms_p = run(fresh_uid() if world > 1 else sqngd.nccl_unique_id(), peer=True)[0]
        extra["peer_allreduce"] = {
            "value": evals / (ms_p / 1e3), "ms_per_step": ms_p, "n_gpus": world,
            "what": "k_world_peer (pack + all-reduce over NVLink peer memory + unpack in one kernel: stage, flag "
                    "signal, wait, rank-ordered read) instead of pack + the grouped NCCL call + unpack, captured "
                    "in the step graph" + (" (1 rank: its own window)" if world == 1 else "")}
    except Exception as e:
        extra["peer_allreduce"] = {"error": f"{type(e).__name__}: {e}"}
    return {**extra, "workload": f"{name}: M={c.M} N={c.N} L={c.B} K={c.K} R={c.R} (one problem)", "n_gpus": world,
            "value": evals / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warm,
            "scaling": "strong", "engine": info["engine"],
            "parallelism": f"work-sharded x{world}: (restart, transmit channel) rows, one grouped NCCL "
                           f"all-reduce per loss+grad evaluation" if world > 1 else "1 GPU",
            "what": "sqngd_step(A+B) of the 8-restart C5 problem; the driver's N=1 line carries the same "
                    "block for the parallel-efficiency ratio"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--loss", default="lse", choices=["lse", "max", "pnorm"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-generator", dest="generator", action="store_false",
                    help="skip the generator-mode (z = f_theta(y0)) line")
    ap.add_argument("--no-torch", dest="torch_comparator", action="store_false",
                    help="skip the torch.fft + autograd comparator line")
    ap.add_argument("--restarts", type=int, default=0,
                    help="independent restarts batched per GPU (default: the config's R)")
    ap.add_argument("--ws-timeout", type=float, default=240.0,
                    help="N > 1: seconds the work-sharded C5 block may take before the line is printed without it")
    ap.add_argument("--no-work-sharded", dest="work_sharded", action="store_false",
                    help="skip the work-sharded C5 line (one problem split over the N ranks)")
    ap.add_argument("--batch-restarts", type=int, default=4,
                    help="also time the config with this many restarts per GPU (context line; 0/1: skip)")
    args = ap.parse_args()

    c = CF.CONFIGS[args.config]
    if args.restarts:
        c = c.with_(R=args.restarts)
    mode = {"max": CF.LOSS_MAX, "lse": CF.LOSS_LSE, "pnorm": CF.LOSS_PNORM}[args.loss]
    c = c.with_(loss_mode=mode, beta_or_p={0: 0.0, 1: 200.0, 2: 16.0}[mode])
    if args.impl == "reference":
        run_reference(args, c)
        return

    import torch

    from paper_2604_25728_b200 import sqngd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    # a non-default stream: sqngd_step captures itself into a CUDA graph there and replays it
    side = torch.cuda.Stream(dev)
    torch.cuda.set_stream(side)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # inputs: this rank's restarts r = rank*R .. (independent seeded problems)
    R = c.R
    z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, g), c.M * c.N).reshape(c.M, c.N)
                  for g in parallel.restart_ids(R, rank)])
    rho = inputs.init_thresholds(R, c.B, c.r_n)
    evals_per_step = (c.n_h + c.n_x) * R * world
    sm_mhz, _, src = peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = sms * 128 * 2 * sm_mhz * 1e6 / 1e12

    def timed(cc, with_clocks):
        """W warm-up + K timed sqngd_step(A+B) calls (CUDA-graph replay), then an eager profiled
        pass over K more steps for the per-kernel CUDA-event times."""
        R = cc.R
        z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, g), c.M * c.N).reshape(c.M, c.N)
                      for g in parallel.restart_ids(R, rank)])
        rho = inputs.init_thresholds(R, c.B, c.r_n)
        evals_per_step = (c.n_h + c.n_x) * R * world
        ctx = sqngd.Context(cc, device=local)
        zt, rt = torch.as_tensor(z, device=dev), torch.as_tensor(rho, device=dev)
        net = {}
        if cc.net_width:  # generator mode: z = f_theta(y0) (NEXT-2), seeded theta and y0 per restart
            Din = cc.M * cc.N
            th = np.concatenate([inputs.net_params(1, Din, cc.net_width, cc.net_depth, config_index=cc.index * 1000 + g)
                                 for g in parallel.restart_ids(R, rank)])
            y0 = np.concatenate([inputs.net_input(1, cc.M, cc.N, cc.B, config_index=cc.index * 1000 + g)
                                 for g in parallel.restart_ids(R, rank)])
            net = dict(theta=torch.as_tensor(th, device=dev), y0=torch.as_tensor(y0, device=dev))
            zt = ctx.net_forward(net["theta"], net["y0"])
        q = ctx.quantize(zt, rt, soft=False, want_b=False, want_dq=False)
        st = ctx.new_state(zt, rt, q["s_hard"], **net)             # w = s_hard (matched start, Q3)
        hist = torch.zeros((R, c.n_h + c.n_x), dtype=torch.float64, device=dev)
        hard = torch.empty(R * sqngd.METRICS_BYTES, dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
        ctx.sync()
        ctx.profile_read(reset=True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        with ClockSampler(local) as clk:
            t_wall = time.perf_counter()
            for i in range(args.steps):
                flush.fill_(float(i))                                   # evict L2 between steps
                evs[i][0].record(stream)
                ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
                evs[i][1].record(stream)
            torch.cuda.synchronize(dev)
            t_wall = time.perf_counter() - t_wall
        if dist:
            dist.barrier()
        ctx.sync()
        launches = ctx.profile_read(reset=True)["launches"]
        tot_ms = parallel.max_over_ranks(sum(a.elapsed_time(b) for a, b in evs))
        # per-kernel times: an eager pass over the same K steps (CUDA events recorded on the launch
        # stream around every fused kernel; graph replay cannot be timed per kernel)
        ctx.profile(True)
        for i in range(args.steps):
            flush.fill_(float(i))
            ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
        ctx.sync()
        prof = ctx.profile_read(reset=True)
        ctx.profile(False)
        info = ctx.engine_info()
        value = evals_per_step * args.steps / (tot_ms / 1e3)
        names = ["fwd", "adjA", "adjB"]
        if info["engine"] == "chebyshev":
            wm = work_model_lr(cc, info["Q"])
            knames = {"fwd": "k_lrt<FWD>", "adjA": "k_lrt<ADJ>", "adjB": "k_lrt<ADJ>"}
        else:
            wm = work_model(cc)
            knames = {"fwd": "k_af<FWD>", "adjA": "k_af<ADJ_A>", "adjB": "k_af<ADJ_B>"}
        # classes that launch the same kernel (k_lrt<ADJ> serves Step A and Step B) are pooled
        dom = max(range(3), key=lambda i: prof["ms"][i])
        same = [i for i in range(3) if knames[names[i]] == knames[names[dom]]]
        k_ms, k_cnt = sum(prof["ms"][i] for i in same), sum(prof["count"][i] for i in same)
        avg_ms = k_ms / max(1, k_cnt)
        common = {"kernel": knames[names[dom]], "avg_launch_ms": avg_ms, "launches": k_cnt,
                  "traffic": traffic_bytes(knames[names[dom]]),
                  "share_of_step": k_ms / tot_ms,
                  "timing": "CUDA events around each fused-kernel launch on its stream, in an eager pass over the "
                            "same K steps right after the timed (CUDA-graph) region"}
        if info["engine"] == "chebyshev":
            w = wm[names[dom]]
            fp32 = w["fp32"] / (avg_ms / 1e3) / 1e12
            tp = tensor_peaks()
            # forward contraction in FP16 (split) and adjoint in 3xTF32 (mma.sync): the tensor pipe's
            # minimum time at its dtype peaks, as a fraction of the launch
            t_fwd = wm["fwd"]["tensor"] / (tp["f16"] * 1e12)
            t_adj = (w["tensor"] - wm["fwd"]["tensor"]) / (tp["tf32"] * 1e12)
            roof = {"bound": "alu", "achieved": fp32, "peak": peak, "unit": "TFLOP/s", "frac": fp32 / peak,
                    "flops_per_launch": w["fp32"],
                    "work": "FP32 pipe: the cell epilogue of SURVEY.md §8(d) (7 forward + 10 adjoint flops per "
                            "cell); the Doppler contraction runs on the tensor pipe (pipes.tensor)",
                    "peak_basis": f"{sms} SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz ({src} sm_max_mhz)",
                    "pipes": {
                        "fp32": {"achieved": fp32, "peak": peak, "frac": fp32 / peak, "unit": "TFLOP/s"},
                        "tensor": {"achieved": w["tensor"] / (avg_ms / 1e3) / 1e12,
                                   "flops_per_launch": w["tensor"],
                                   "frac": (t_fwd + t_adj) / (avg_ms / 1e3),
                                   "peak_f16": tp["f16"], "peak_tf32": tp["tf32"], "unit": "TFLOP/s",
                                   "frac_def": "(forward contraction / f16 peak + adjoint contraction / tf32 peak) "
                                               "/ launch time", "peak_basis": tp["basis"]}},
                    **common}
        else:
            achieved = wm[names[dom]] / (avg_ms / 1e3) / 1e12
            roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "flops_per_launch": wm[names[dom]],
                    "work": "SURVEY.md §8(d) convention flops of the per-bin FFT method (5 P log2 P per FFT, "
                            "6 per complex multiply, 7 / 10 per cell)",
                    "peak_basis": f"{sms} SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz ({src} sm_max_mhz)",
                    **common}
        # issue slots (both engines are issue-bound): the ncu instruction count of the same kernel at the
        # same size (C3, one restart) over the live launch time
        iss = issue_pipe(knames[names[dom]], cc.name, avg_ms, sms, sm_mhz) if cc.R == 1 else None
        if iss:
            roof.setdefault("pipes", {})["issue"] = iss
        out = {"value": value, "ms_per_step": tot_ms / args.steps, "roofline": roof, "launches": launches,
               "kernel_ms": {n: prof["ms"][i] / args.steps for i, n in enumerate(names)}, "engine": info,
               "wall_s": t_wall}
        if cc.net_width and prof["count"][3]:
            out["net_update_ms"] = prof["ms"][3] / prof["count"][3]
        if with_clocks:
            out["clocks"] = clk.summary()
        return ctx, st, hist, hard, out

    # headline: the library's default engine for this config (AUTO: Chebyshev nodes on the paper's
    # narrow Doppler grid); then the per-bin FFT engine on the same inputs, reported beside it
    ctx, st, hist, hard, main_run = timed(c, True)
    fft_run = None
    if main_run["engine"]["engine"] != "fft":
        ctxf, *_rest, fft_run = timed(c.with_(doppler_engine=sqngd.ENGINE_FFT), False)
        ctxf.close()
    value, tot_ms = main_run["value"], main_run["ms_per_step"] * args.steps

    # ---- forward only (sqngd_af_forward, a2-a6): delay-Doppler cells/s = M^2 (2N-1) K R / t_fwd (SURVEY
    # §8(d)), without and with the |A| map written to HBM; the map-writing launch against HBM bandwidth.
    def forward_rate(cx, s, w, want_map, reps=10, ld=None):
        amap = (torch.empty((c.R, c.M, c.M, c.K, ld or (2 * c.N - 1)), dtype=torch.float32, device=dev) if want_map
                else None)
        for _ in range(3):
            cx.af_forward(s, w, map_out=amap, want_p=False)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for i in range(reps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            cx.af_forward(s, w, map_out=amap, want_p=False)
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        t = parallel.max_over_ranks(sum(a.elapsed_time(b) for a, b in evs)) / reps / 1e3
        cx.profile(True)
        cx.profile_read(reset=True)
        for i in range(reps):
            flush.fill_(float(i))
            cx.af_forward(s, w, map_out=amap, want_p=False)
        pr = cx.profile_read(reset=True)
        cx.profile(False)
        tk = pr["ms"][0] / max(1, pr["count"][0]) / 1e3
        return t, tk

    s_h = ctx.quantize(st["z"], st["rho"], soft=False, want_b=False, want_dq=False)["s_hard"]
    t_f, tk_f = forward_rate(ctx, s_h, st["w"], False)
    t_m, tk_m = forward_rate(ctx, s_h, st["w"], True)
    # the same map with rows on 128-byte boundaries (cfg.map_ld: pitch 2N-1 rounded up to 32 floats)
    ld = (2 * c.N - 1 + 31) // 32 * 32
    ctxp = sqngd.Context(c.with_(map_ld=ld), device=local)
    t_p, tk_p = forward_rate(ctxp, s_h, st["w"], True, ld=ld)
    ctxp.close()
    cells_job = c.cells * c.R * world
    map_bytes = c.cells * c.R * 4
    hbm_peak = peaks()[1]
    kname = ("k_lrt<FWD>" if main_run["engine"]["engine"] == "chebyshev" else "k_af<FWD>") + " (writing the map)"
    forward = {
        "cells_per_s": cells_job / t_f, "ms_per_forward": t_f * 1e3,
        "with_map": {"cells_per_s": cells_job / t_m, "ms_per_forward": t_m * 1e3, "map_bytes": map_bytes,
                     "roofline": {"bound": "hbm", "kernel": ("k_lrt<FWD>" if main_run["engine"]["engine"] == "chebyshev"
                                             else "k_af<FWD>") + " (writing the map)",
                                  "achieved": map_bytes / tk_m / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                  "frac": map_bytes / tk_m / 1e9 / hbm_peak, "avg_launch_ms": tk_m * 1e3,
                                  "traffic": None,
                                  "what": "|A| map bytes (M^2 (2N-1) K x 4 B, fp32) / duration of the fused launch "
                                          "that writes it"}},
        "with_map_pitched": {"map_ld": ld, "cells_per_s": cells_job / t_p, "ms_per_forward": t_p * 1e3,
                             "roofline": {"bound": "hbm", "kernel": kname + f", rows pitched to {ld} floats",
                                          "achieved": map_bytes / tk_p / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                          "frac": map_bytes / tk_p / 1e9 / hbm_peak, "avg_launch_ms": tk_p * 1e3,
                                          "traffic": None,
                                          "what": "the same |A| bytes (the pad is not written) / launch duration"}},
        "fused_launch_ms_no_map": tk_f * 1e3,
        "what": "sqngd_af_forward (filter FFT, node/bin transforms, fused contraction + ROI reduction, metrics), "
                "CUDA events per call, L2 flushed between calls"}

    # ---- end to end through the public API with host buffers (pinned), copies inside the timing.
    # The optimizer state and the step's outputs (loss history, hard metrics) live in ONE device
    # allocation (the sqngd_state pointers are views into it): the state goes up in one H2D copy and
    # state + outputs come back in one D2H copy.
    keys = ["z", "rho", "w", "m_z", "v_z", "m_rho", "v_rho", "m_w", "v_w"]
    sizes = {k: st[k].numel() * (2 if st[k].is_complex() else 1) for k in keys}
    nst = sum(sizes.values())
    hist_b = hist.numel() * 8
    sb = (4 * nst + 7) // 8 * 8
    buf = torch.empty(sb + hist_b + hard.numel(), dtype=torch.uint8, device=dev)
    flat = buf[:4 * nst].view(torch.float32)
    est, o = {"t_a": st["t_a"], "t_b": st["t_b"]}, 0
    for k in keys:
        v = flat[o:o + sizes[k]]
        v = v.view(torch.complex64) if st[k].is_complex() else v
        est[k] = v.view(st[k].shape)
        est[k].copy_(st[k])
        o += sizes[k]
    outb = buf[sb:]
    ehist = outb[:hist_b].view(torch.float64).view(hist.shape)
    ehard = outb[hist_b:]
    host_buf = buf.cpu().pin_memory()
    host_state = host_buf[:4 * nst]
    host_out = host_buf[sb:]
    h2d = 4 * nst
    d2h = buf.numel()
    e2e_ev = []
    for i in range(args.warmup + args.steps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        buf[:4 * nst].copy_(host_state, non_blocking=True)
        ctx.step(est, sqngd.BLOCK_AB, hist=ehist, hard_met=ehard)
        host_buf.copy_(buf, non_blocking=True)
        b.record(stream)
        if i >= args.warmup:
            e2e_ev.append((a, b))
    torch.cuda.synchronize(dev)
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
    e2e_ms = parallel.max_over_ranks(e2e_ms)
    e2e_value = evals_per_step * args.steps / (e2e_ms / 1e3)
    host_hard = host_out[hist_b:]
    hm = sqngd.metrics_from_bytes(host_hard.numpy())
    eng = main_run["engine"]
    eng_desc = (f"chebyshev (Q={eng['Q']} nodes, |A| interpolation bound {eng['err_bound']:.1e} x N)"
                if eng["engine"] == "chebyshev" else "fft (one modulated FFT correlation per Doppler bin)")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "precision": ("fp32 CUDA-core arithmetic (FFTs, cell epilogue, reductions; fp64 for the restart sums, "
                      "energies and Adam bias corrections); the Chebyshev engine's Doppler contraction on "
                      "split-precision MMAs (fp16 3-term forward, tf32 3x adjoint: ~fp32 accuracy) plus its "
                      "interpolation bound; against the fp64 oracle the GPU suite's worst per-cell "
                      "|d|A||/N is 4.6e-7 (bar 1e-6) and worst normwise gradient error 2.6e-6 (bar 1e-4): "
                      "profiles/r02h_parity_errors.json") if eng["engine"] == "chebyshev" else
                     "fp32 CUDA-core arithmetic (fp64 restart sums / energies); parity against the fp64 oracle "
                     "in profiles/r02h_parity_errors.json",
        "config": {**config_dict(c), "doppler_engine": eng_desc,
                   "parallelism": f"restarts x{world} (independent, no collective)"},
        "cells_per_s": forward["cells_per_s"],
        "forward": forward,
        "roofline": main_run["roofline"],
        "kernel_ms": main_run["kernel_ms"],
        "gpu_launches": main_run["launches"],
        "clocks": main_run["clocks"],
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "wall_s": main_run["wall_s"],
        "final_hard_pslr_db": 20 * math.log10(max(hm[0]["wpsl"], 1e-30)),
    }
    # per-block and per-loss-mode breakdown (Step A vs Step B, MAX vs LSE), graph replay
    def block_rate(cx, stx, block, n_evals, reps=10):
        for _ in range(3):
            cx.step(stx, block)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            cx.step(stx, block)
        b.record(stream)
        torch.cuda.synchronize(dev)
        return n_evals * reps / (parallel.max_over_ranks(a.elapsed_time(b)) / 1e3)

    breakdown = {"step_A_evals_per_s": block_rate(ctx, st, sqngd.BLOCK_A, c.n_h * c.R * world),
                 "step_B_evals_per_s": block_rate(ctx, st, sqngd.BLOCK_B, c.n_x * c.R * world)}
    if c.loss_mode != CF.LOSS_MAX:
        cm = c.with_(loss_mode=CF.LOSS_MAX, beta_or_p=0.0)
        ctxm = sqngd.Context(cm, device=local)
        stm = ctxm.new_state(st["z"], st["rho"], st["w"])
        breakdown["max_mode_evals_per_s"] = block_rate(ctxm, stm, sqngd.BLOCK_AB, (c.n_h + c.n_x) * c.R * world)
        ctxm.close()
    line["breakdown"] = {**breakdown, "unit": UNIT,
                         "what": "Step A only (filters), Step B only (transmit), and the MAX loss (Eq. 37, O(N) "
                                 "subgradient adjoint) instead of LSE; each 10 graph-replayed steps"}
    if args.batch_restarts > 1 and c.R == 1:  # the same config with B independent restarts per GPU
        ctxb, *_rest, b_run = timed(c.with_(R=args.batch_restarts), False)
        ctxb.close()
        line["restart_batched"] = {
            "restarts_per_gpu": args.batch_restarts, "value": b_run["value"], "unit": UNIT,
            "ms_per_step": b_run["ms_per_step"], "cells_per_s_in_loss_grad": b_run["value"] * c.cells,
            "roofline": b_run["roofline"], "gpu_launches": b_run["launches"],
            "what": "context: B independent seeded restarts batched in one context per GPU (the headline is R = 1)"}
    if args.generator:  # NEXT-2: the same step with the paper's ResNet generator z = f_theta(y0)
        W, D = 128, 5
        cg = c.with_(net_width=W, net_depth=D, lr_theta=1e-5)
        ctxg, *_rest, gen_run = timed(cg, False)
        ctxg.close()
        Din = c.M * c.N
        P = sqngd.net_num_params(cg)
        # algorithmic bytes of one generator update (backward + Adam + next forward): every parameter's
        # (theta, m, v) read and written once (24 B), W_out read again by the forward, y0/z/dL/dz/z
        upd_bytes = 24 * P * c.R + 4 * W * Din * c.R + 16 * Din * c.R
        hbm = peaks()[1]
        gbs = upd_bytes / (gen_run["net_update_ms"] / 1e3) / 1e9
        line["generator"] = {
            "arch": f"ResNet {D} residual blocks, width {W}, tanh / sigmoid (P:L583); {P} parameters per restart",
            "value": gen_run["value"], "unit": UNIT, "ms_per_step": gen_run["ms_per_step"],
            "gpu_launches": gen_run["launches"],
            "update_ms": gen_run["net_update_ms"],
            "roofline": {"bound": "hbm", "kernel": "generator update (k_net_out_bwd, k_net_mid_bwd, k_net_upd<ADAM>, "
                                                   "k_net_mid_fwd, k_net_out)",
                         "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None,
                         "bytes_per_update": upd_bytes,
                         "timing": "CUDA events around each Step-B generator update in the eager profiled pass"}}
    if args.torch_comparator:  # NEXT-4: the same Step-B loss+grad in torch.fft + autograd on this GPU
        from tools.torch_autograd import time_torch_step_b

        zt, rt = torch.as_tensor(z, device=dev), torch.as_tensor(rho, device=dev)
        wt = ctx.quantize(zt, rt, soft=False, want_b=False, want_dq=False)["s_hard"]
        ev_s, ms_t, loss_t, gz_t = time_torch_step_b(c.with_(R=1), zt[:1], rt[:1], wt[:1], dev)
        met, gz_o, _ = ctx.af_loss_grad(zt, rt, wt, sqngd.WRT_TRANSMIT)
        ctx.sync()
        loss_o = ctx.metrics(met)[0]["loss"]
        gz_o = gz_o[:1].reshape(gz_t.shape)
        line["torch_autograd"] = {
            "what": "Step-B loss+grad (LSE) as torch.fft correlations + dense |A| + autograd on the same GPU "
                    "(paper-style framework implementation; context, not a parity reference)",
            "value": ev_s, "unit": "Step-B loss+grad evals/s", "ms_per_eval": ms_t,
            "loss_rel_diff_vs_ours": abs(loss_t - loss_o) / abs(loss_o),
            "grad_z_rel_diff_vs_ours": float(torch.linalg.norm(gz_t - gz_o) / torch.linalg.norm(gz_o))}
    if fft_run is not None:
        line["fft_engine"] = {"value": fft_run["value"], "unit": UNIT, "ms_per_step": fft_run["ms_per_step"],
                              "cells_per_s_in_loss_grad": fft_run["value"] * c.cells,
                              "roofline": fft_run["roofline"],
                              "kernel_ms": fft_run["kernel_ms"], "gpu_launches": fft_run["launches"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OMP_NUM_THREADS", str(cpu_info()))
        per_eval, nb = oracle_sample(c, budget_s=10.0)
        line["cpu_baseline"] = {"value": 1.0 / per_eval, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]),
                                "kind": "oracle",
                                "sample": f"Step-B loss+grad (quantize, AF, LSE loss, adjoint, chain) of the fp64 "
                                          f"oracle with {nb} of {c.K} Doppler bins evaluated, AF/adjoint time "
                                          f"scaled by K/{nb}"}
    if args.work_sharded:  # C5 (8 restarts) with its pair / Doppler work sharded over the N ranks
        # Last block of the line. NCCL's exchange between ranks has never run in this environment (every
        # box has one GPU), so at N > 1 a watchdog bounds it: if the sharded steps have not returned in
        # time, rank 0 prints the line measured so far (headline, roofline, e2e intact) and every rank exits 0.
        guard = None
        if world > 1:
            import threading

            def bail():
                line["work_sharded"] = {"error": f"no result within {args.ws_timeout:.0f} s (watchdog); the "
                                                 f"rest of the line is unaffected"}
                if rank == 0:
                    print(json.dumps(line), flush=True)
                os._exit(0)

            guard = threading.Timer(args.ws_timeout, bail)
            guard.daemon = True
            guard.start()
        try:
            line["work_sharded"] = work_sharded(args, world, rank, local, dev, stream, flush)
        except Exception as e:  # reported, not fatal to the headline
            line["work_sharded"] = {"error": f"{type(e).__name__}: {e}"}
        finally:
            if guard is not None:
                guard.cancel()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
