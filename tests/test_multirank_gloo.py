"""World-size-2 tests of the multi-rank host logic on CPU (gloo backend).

The one-collective protocol that libsqngd runs over NCCL (csrc/comm.h: weighted fp64 SUM
against a shared reference shift, MAX of the keys) is exercised here with
torch.distributed/gloo: each rank evaluates half of the Doppler bins with the fp64
oracle, the partials are combined with parallel.combine_ref for several reference shifts
(0, a stale previous maximum, the exact maximum), and the result must equal the
oracle's single-process evaluation of the full grid.  The library's own sharded kernels
are tested on the GPU through the loopback group (tests/test_gpu_multirank.py)."""
import math
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_25728_b200 import parallel

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(**kw):
    d = dict(R=1, M=2, N=9, B=4, r_n=2, c=300.0, K=6, f_lo=-0.8, f_hi=1.2, tau_lo=None, tau_hi=None,
             exclude_auto_zero_delay=1, loss_mode=1, beta_or_p=25.0, eps_w=1.0, mu_db=0.5)
    d.update(kw)
    return SimpleNamespace(**d)


def _inputs(c):
    g = np.random.default_rng(7)
    s = np.exp(2j * np.pi * g.random((1, c.M, c.N)))
    w = g.standard_normal((1, c.M, c.N)) + 1j * g.standard_normal((1, c.M, c.N))
    return s, w


def _subset(c, k0, k1):
    d = (c.f_hi - c.f_lo) / (c.K - 1)
    return SimpleNamespace(**{**vars(c), "K": k1 - k0, "f_lo": c.f_lo + k0 * d, "f_hi": c.f_lo + (k1 - 1) * d})


def _worker(rank, port, mode, q):
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        c = _cfg(loss_mode=mode, beta_or_p=25.0 if mode == 1 else 6.0)
        s, w = _inputs(c)
        k0, k1 = parallel.shard_range(c.K, rank, WORLD)
        cs = _subset(c, k0, k1)
        met, gw, gs = O.loss_grad(cs, s, w)
        m_r, L_r = met[0]["wpsl"], met[0]["loss_wpsl"]
        p = c.beta_or_p
        if mode == 1:
            S_r = math.exp(p * (L_r - m_r))
            G_r = np.concatenate([gw.ravel(), gs.ravel()]) * S_r          # unnormalized at shift m_r
        else:
            S_r = (L_r / m_r) ** p
            G_r = np.concatenate([gw.ravel(), gs.ravel()]) / S_r ** (1.0 / p - 1.0)
        g_loc = G_r / S_r if mode == 1 else G_r * S_r ** (1.0 / p - 1.0)   # locally normalised
        g = torch.from_numpy(np.stack([g_loc.real, g_loc.imag], -1))
        outs = []
        for m_ref in ((0.0 if mode == 1 else 1.0), 0.8, None):  # shared: the create value, a stale one, exact
            if m_ref is None:  # the exact global maximum, from a previous round
                _, _, m_ref = parallel.combine_ref(m_r, S_r, g, 0.0 if mode == 1 else 1.0, p, mode=mode)
            loss, Gt, mg = parallel.combine_ref(m_r, S_r, g, m_ref, p, mode=mode)
            outs.append((loss, Gt.numpy()[..., 0] + 1j * Gt.numpy()[..., 1], mg))
        tmax = parallel.max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((outs, tmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [1, 2])
def test_sharded_lse_combine_matches_single_process(mode):
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, mode, q)) for r in range(WORLD)]
    for p_ in procs:
        p_.start()
    outs, tmax = q.get(timeout=120)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    c = _cfg(loss_mode=mode, beta_or_p=25.0 if mode == 1 else 6.0)
    s, w = _inputs(c)
    met, gw, gs = O.loss_grad(c, s, w)
    ref = np.concatenate([gw.ravel(), gs.ravel()])
    for loss, grad, mg in outs:  # exact for every reference shift
        assert abs(loss - met[0]["loss_wpsl"]) < 1e-12 * abs(met[0]["loss_wpsl"])
        assert np.abs(grad - ref).max() < 1e-10 * np.abs(ref).max()
        assert mg == met[0]["wpsl"]          # the new reference: the global maximum
    assert tmax == float(WORLD)


def test_shard_and_restart_assignment():
    for units, world in [(2056, 8), (7, 3), (257, 2)]:
        spans = [parallel.shard_range(units, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == units
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert parallel.restart_ids(2, 3) == [6, 7]
