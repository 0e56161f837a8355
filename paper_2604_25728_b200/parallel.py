"""Multi-rank host logic shared by bench.py and the tests.

Two ways the hot path spans GPUs:

* independent restarts (bench.py --gpus N, "weak"): rank r optimizes its own seeded
  restarts, no data-path collective; only the timing is reduced (max over ranks);
* one problem sharded over ranks (the library's world > 1 mode): each rank evaluates a
  shard (FFT engine: a slice of the (restart, channel, bin) units; Chebyshev engine: a
  slice of the (restart, transmit channel) rows) and ONE grouped collective per
  evaluation combines the per-restart partials against a reference shift every rank
  holds (csrc/comm.h, misc_kernels.cuh k_world_pack / k_world_unpack).  `combine_ref`
  below restates that arithmetic over torch.distributed so the protocol is testable
  with gloo on CPU (gloo has no grouped call: the SUM and the MAX are two calls there).
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


def combine_ref(m, S, g, m_ref: float, beta: float, mode: int = 1, group=None):
    """One restart's combine of the library's world > 1 protocol (csrc/comm.h).

    m: the rank's shift (-inf if it has no cells); S: its sum of phi at that shift; g: its
    gradient normalised locally (LSE: G / S, p-norm: G S^{1/p - 1}) as a float64 tensor; m_ref: the
    reference shift, identical on every rank.  Weights (fp64):
      LSE:    wS = wG = e^{beta (m - m_ref)} S
      p-norm: wS = (m / m_ref)^p S,  wG = (m / m_ref)^{p-1} S^{1 - 1/p}
    SUM of [wS | wG g] and MAX of m over ranks, then
      LSE:    loss = m_ref + ln(sum wS) / beta,   grad = sum(wG g) / sum wS
      p-norm: loss = m_ref (sum wS)^{1/p},        grad = sum(wG g) (sum wS)^{1/p - 1}
    Returns (loss, grad, new m_ref = max over ranks of m)."""
    import torch
    import torch.distributed as dist

    if not (S > 0) or m == -math.inf:
        wS = wG = 0.0
    elif mode == 1:
        wS = wG = math.exp(beta * (m - m_ref)) * S
    else:
        rho = m / m_ref
        wS = rho ** beta * S
        wG = rho ** (beta - 1.0) * S ** (1.0 - 1.0 / beta)
    pay = torch.cat([torch.tensor([wS], dtype=torch.float64), (g.to(torch.float64) * wG).reshape(-1)])
    mx = torch.tensor([m if m > -math.inf else -1.0], dtype=torch.float64)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(pay, group=group)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    St, Gt = float(pay[0]), pay[1:].reshape(g.shape)
    if mode == 1:
        loss, grad = m_ref + math.log(St) / beta, Gt / St
    else:
        loss, grad = m_ref * St ** (1.0 / beta), Gt * St ** (1.0 / beta - 1.0)
    return loss, grad, float(mx.item())
