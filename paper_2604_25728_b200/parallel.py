"""Multi-rank host logic shared by bench.py and the tests.

Two ways the hot path spans GPUs:

* independent restarts (bench.py --gpus N, "weak"): rank r optimizes its own seeded
  restarts, no data-path collective; only the timing is reduced (max over ranks);
* one problem sharded over ranks (the library's world > 1 mode): each rank evaluates a
  contiguous slice of the (restart, channel, Doppler) units and the per-restart
  partials are combined by the max-then-sum protocol below.  libsqngd implements it
  with NCCL (csrc/comm.h: k_red_pack / k_red_rescale / k_red_unpack); `combine_lse`
  is the same arithmetic over torch.distributed so it is testable with gloo on CPU.
"""
from __future__ import annotations

import math


def shard_range(units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of `units` owned by `rank` (mirrors sqngd_shard_range)."""
    world = max(1, world)
    base, rem = divmod(units, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def restart_ids(r_per_rank: int, rank: int) -> list[int]:
    """Global restart indices owned by `rank` when every rank runs r_per_rank restarts."""
    return [rank * r_per_rank + i for i in range(r_per_rank)]


def max_over_ranks(x: float, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(x)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def combine_lse(m, S, G, beta: float, mode: int = 1, group=None):
    """Combine per-rank LSE / p-norm partials of one restart.

    m: the rank's shift (max v over its cells, -inf if none); S: sum of phi at that shift;
    G: the rank's unnormalized gradient (sum of phi-weighted cotangent contributions) at
    that shift (a tensor).  Returns (m_global, S_global, G_global) at the global shift:
      1. all-reduce MAX of m;  2. rescale S and G to it;  3. all-reduce SUM of S and G.
    LSE: phi = e^{beta (v - m)}, rescale e^{beta (m_r - m)} for both S and G;
    PNORM: phi = (v/m)^p, S rescales by (m_r/m)^p and G (weights (v/m)^{p-1}) by (m_r/m)^{p-1}.
    """
    import torch
    import torch.distributed as dist

    mt = torch.tensor([float(m)], dtype=torch.float64, device=G.device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(mt, op=dist.ReduceOp.MAX, group=group)
    mg = float(mt.item())
    if not (S > 0) or m == -math.inf:
        sc_S = sc_G = 0.0
    elif mode == 1:
        sc_S = sc_G = math.exp(beta * (m - mg))
    else:
        sc_S = (m / mg) ** beta
        sc_G = (m / mg) ** (beta - 1.0)
    St = torch.tensor([S * sc_S], dtype=torch.float64, device=G.device)
    Gt = (G * sc_G).to(torch.float64)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(St, group=group)
        dist.all_reduce(Gt, group=group)
    return mg, float(St.item()), Gt
