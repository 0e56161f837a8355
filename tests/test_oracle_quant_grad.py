"""Pins of the oracle's quantizer (Eqs. 21-25, 43) and of every gradient
(finite differences of the oracle's own loss), plus Adam / projections."""
import math
import os
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def cfg(**kw):
    d = dict(R=1, M=2, N=5, B=4, r_n=1, c=300.0, K=3, f_lo=-0.5, f_hi=0.5, tau_lo=None, tau_hi=None,
             exclude_auto_zero_delay=1, loss_mode=1, beta_or_p=20.0, eps_w=0.4, mu_db=0.5,
             lr_w=5e-2, lr_z=1e-4, adam_b1=0.9, adam_b2=0.999, adam_eps=1e-8, n_h=2, n_x=2)
    d.update(kw)
    return SimpleNamespace(**d)


def init_rho(B, r_n):
    return (np.arange(B * r_n) + 0.5) / (B * r_n)


def rnd(shape, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


# ------------------------------------------------------------------ quantizer
def test_eq25_level_set():
    lines = [l for l in open(os.path.join(GOLD, "eq25_levelset.txt")) if not l.startswith("#")]
    B, r_n, c = [float(x) for x in lines[0].split()]
    want = sorted(float(x) for x in lines[1].split())
    B, r_n = int(B), int(r_n)
    rho = init_rho(B, r_n)
    zs = np.linspace(-0.05, 1.05, 4001)
    levels = sorted({O.QR_level(B, r_n, c, rho, z) / B for z in zs})
    assert levels == want
    # and the phase indices are the QPSK alphabet
    q = O.quantize(cfg(R=1, M=1, N=len(zs), B=B, r_n=r_n, c=c), zs.reshape(1, 1, -1), rho.reshape(1, -1))
    assert set(np.unique(q["b_hard"])) == {0, 1, 2, 3}
    np.testing.assert_allclose(np.abs(q["s_hard"]), 1.0, atol=1e-15)
    np.testing.assert_allclose(q["s_hard"], np.exp(2j * np.pi * q["b_hard"] / B), atol=1e-15)


def test_soft_quantizer_examples_and_bounds():
    rho = init_rho(4, 1)
    assert abs(O.QA(4, 1, 300.0, rho, 0.25) - 0.25) < 1e-6
    assert O.QA(4, 1, 300.0, rho, -10.0) < 1e-12                 # z -> -inf
    # Sum 2 a_i = r_n at z -> +inf
    assert abs(O.QA(8, 3, 300.0, init_rho(8, 3), 10.0) - 3.0) < 1e-12
    # monotone, and |Q_A'| <= c r_n / 2
    B, r_n, c = 8, 5, 300.0
    rho = init_rho(B, r_n)
    zs = np.linspace(-0.1, 1.1, 1500)
    ys = np.array([O.QA(B, r_n, c, rho, z) for z in zs])
    assert np.all(np.diff(ys) >= 0)                              # saturates to flat in fp64 outside
    inner = (zs > 0.01) & (zs < 0.99)
    assert np.all(np.diff(ys[inner]) > 0)
    d = [O.dQA(B, r_n, c, rho, z) for z in zs]
    assert max(d) <= c * r_n / 2 + 1e-9 and min(d) > 0


def test_dQA_finite_difference():
    B, r_n, c = 4, 3, 40.0
    rho = init_rho(B, r_n) + 0.01 * np.sin(np.arange(B * r_n))
    for z in (0.03, 0.31, 0.5, 0.77):
        h = 1e-6
        fd = (O.QA(B, r_n, c, rho, z + h) - O.QA(B, r_n, c, rho, z - h)) / (2 * h)
        assert abs(fd - O.dQA(B, r_n, c, rho, z)) < 1e-6 * max(1, abs(fd))


def test_hard_quantizer_branches():
    B, r_n, c = 4, 3, 300.0
    rho = init_rho(B, r_n)
    assert O.QR_level(B, r_n, c, rho, rho[0] - 1e-9) == 0               # x < rho_0
    assert O.QR_level(B, r_n, c, rho, rho[-1]) == B * r_n                # rho_top <= x -> sum 2a_i
    assert O.QR_level(B, r_n, c, rho, rho[3]) == 4                       # boundary goes up
    # interior plateaus: Q_R(z) = i*/B for the default grid (pairwise tanh cancellation)
    for i in range(1, B * r_n):
        z = 0.5 * (rho[i - 1] + rho[i])
        assert O.QR_level(B, r_n, c, rho, z) == i
    # soft -> hard consistency away from thresholds
    zs = np.array([0.5 * (rho[i] + rho[i + 1]) for i in range(B * r_n - 1)])
    for z in zs:
        assert abs(O.QA(B, r_n, c, rho, z) - O.QR_level(B, r_n, c, rho, z) / B) < 1e-3


def test_default_config_edge_levels_differ_from_istar():
    """with r_n = 100, c = 300, B = 16 the midpoint value snaps to a level
    != i* near the edges, so the hard index is not i* mod B there."""
    B, r_n, c = 16, 100, 300.0
    rho = init_rho(B, r_n)
    diff = [i for i in range(1, B * r_n) if O.QR_level(B, r_n, c, rho, 0.5 * (rho[i - 1] + rho[i])) != i]
    assert len(diff) > 0 and all(i < 10 or i > B * r_n - 10 for i in diff)


# ------------------------------------------------------------------ gradients (FD)
def _loss(c, s, w):
    met, _, _ = O.af(c, s, w)
    return met[0]["loss"]


def _fd_complex(c, s, w, which, idx, h=1e-6):
    """2 dL/dv^* = dL/dRe v + j dL/dIm v by central differences."""
    out = []
    for d in (1.0, 1j):
        sp, sm, wp, wm = s.copy(), s.copy(), w.copy(), w.copy()
        if which == "w":
            wp[idx] += h * d
            wm[idx] -= h * d
        else:
            sp[idx] += h * d
            sm[idx] -= h * d
        out.append((_loss(c, sp, wp) - _loss(c, sm, wm)) / (2 * h))
    return out[0] + 1j * out[1]


@pytest.mark.parametrize("mode,param", [(1, 20.0), (2, 6.0), (0, 0.0)])
def test_gradients_match_finite_differences(mode, param):
    c = cfg(loss_mode=mode, beta_or_p=param, K=3, f_lo=-0.7, f_hi=0.9)
    N, M = c.N, c.M
    s = np.exp(2j * np.pi * np.random.default_rng(3).random((1, M, N)))
    w = rnd((1, M, N), 4) * 0.8
    met, gw, gs = O.loss_grad(c, s, w)
    assert abs(met[0]["loss"] - _loss(c, s, w)) < 1e-15
    gmax = max(np.abs(gw).max(), np.abs(gs).max())
    for m in range(M):
        for n in range(N):
            fdw = _fd_complex(c, s, w, "w", (0, m, n))
            fds = _fd_complex(c, s, w, "s", (0, m, n))
            assert abs(fdw - gw[0, m, n]) < 1e-6 * gmax
            assert abs(fds - 2 * gs[0, m, n]) < 1e-6 * gmax


def test_gradient_zero_when_nothing_upstream():
    """eps = 0 and p_m = p_tar: dL = 0 everywhere."""
    c = cfg(eps_w=0.0, mu_db=0.0)
    s = np.exp(2j * np.pi * np.random.default_rng(5).random((1, 2, 5)))
    _, gw, gs = O.loss_grad(c, s, s)
    assert np.abs(gw).max() < 1e-14 and np.abs(gs).max() < 1e-14


def test_chain_rule_finite_differences():
    c = cfg(B=4, r_n=2, c=30.0, loss_mode=1, beta_or_p=15.0)
    R, M, N = 1, c.M, c.N
    z = np.random.default_rng(6).random((R, M, N))
    rho = (init_rho(4, 2) + 0.02 * np.cos(np.arange(8))).reshape(1, -1)
    w = rnd((1, M, N), 7)

    def L(zz, rr):
        q = O.quantize(c, zz, rr)
        return _loss(c, q["s_soft"], w)

    q = O.quantize(c, z, rho)
    _, _, gs = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz, gr = O.chain(c, z, rho, q["s_soft"], gs)
    h = 1e-6
    scale = max(np.abs(gz).max(), np.abs(gr).max())
    for idx in [(0, 0, 0), (0, 1, 3), (0, 0, 4)]:
        zp, zm = z.copy(), z.copy()
        zp[idx] += h
        zm[idx] -= h
        assert abs((L(zp, rho) - L(zm, rho)) / (2 * h) - gz[idx]) < 1e-6 * scale
    for i in range(8):
        rp, rm = rho.copy(), rho.copy()
        rp[0, i] += h
        rm[0, i] -= h
        assert abs((L(z, rp) - L(z, rm)) / (2 * h) - gr[0, i]) < 1e-6 * scale


# ------------------------------------------------------------------ optimizer pieces
def test_adam_examples():
    g = dict(l.split() for l in open(os.path.join(GOLD, "spec_examples.txt")) if not l.startswith("#"))
    x, m, v = np.array([1.0]), np.zeros(1), np.zeros(1)
    O.adam(x, m, v, 2 * x, 1, 0.1)
    assert abs(x[0] - float(g["adam_first"])) < 1e-7
    for t in range(2, 201):
        O.adam(x, m, v, 2 * x, t, 0.1)
    assert abs(x[0]) < 1e-2
    x2 = np.array([0.3, -2.0])
    m2, v2 = np.zeros(2), np.zeros(2)
    O.adam(x2, m2, v2, np.zeros(2), 1, 0.1)                        # zero gradient: unchanged
    np.testing.assert_array_equal(x2, [0.3, -2.0])


def test_filter_projection():
    w = rnd((3, 6), 8)
    w[1] *= 0
    w[1, 0] = 2 * math.sqrt(6)                                   # ||h||^2 = 4N -> scaled by 1/2
    bad = O.project_filters(w)
    assert bad == 0
    np.testing.assert_allclose(np.sum(np.abs(w) ** 2, axis=1), 6.0, rtol=1e-12)
    assert abs(w[1, 0] - math.sqrt(6)) < 1e-12
    w2 = w.copy()
    O.project_filters(w2)                                        # idempotent
    np.testing.assert_allclose(w2, w, atol=1e-15)
    ph = np.exp(0.7j)
    w3 = rnd((2, 5), 9)
    a = (w3 * ph).copy()
    O.project_filters(a)
    b = w3.copy()
    O.project_filters(b)
    np.testing.assert_allclose(a, b * ph, atol=1e-14)            # commutes with a global phase
    z = np.zeros((1, 4), complex)
    assert O.project_filters(z) == 1


def test_threshold_projection():
    r = np.array([[0.1, 0.3, 0.2, 0.9]])
    O.project_thresholds(r)
    np.testing.assert_allclose(r, [[0.1, 0.2, 0.3, 0.9]])
    r = np.array([[0.2, 1.5, 0.5]])
    O.project_thresholds(r)
    np.testing.assert_allclose(r, [[0.2, 0.5, 1 - 1e-4]])
    r = np.array([[0.5, 0.5, 0.5]])
    O.project_thresholds(r)
    np.testing.assert_allclose(r, [[0.5, 0.5 + 1e-6, 0.5 + 2e-6]], atol=1e-15)
    r2 = r.copy()
    O.project_thresholds(r2)
    np.testing.assert_array_equal(r, r2)                         # idempotent


def test_step_block_isolation_and_feasibility():
    c = cfg(B=4, r_n=2, c=300.0, n_h=2, n_x=2, lr_z=1e-3)
    z = np.random.default_rng(11).random((1, 2, 5))
    rho = init_rho(4, 2).reshape(1, -1)
    q = O.quantize(c, z, rho)
    st = O.new_state(z, rho, q["s_hard"])
    z0, r0 = st["z"].copy(), st["rho"].copy()
    O.step(c, st, block=1)
    np.testing.assert_array_equal(st["z"], z0)
    np.testing.assert_array_equal(st["rho"], r0)
    np.testing.assert_allclose(np.sum(np.abs(st["w"]) ** 2, axis=-1), 5.0, rtol=1e-12)
    w0 = st["w"].copy()
    O.step(c, st, block=2)
    np.testing.assert_array_equal(st["w"], w0)
    assert np.all(np.diff(st["rho"], axis=1) > 0)
    assert st["t_a"] == 2 and st["t_b"] == 2


# ---------------------------------------------------------------- O6 stopping_check pins
# SPEC S:L546-550 stopping_check examples and P:L485 / Alg. 1.
def test_stopping_check_spec_examples():
    T = 12
    improving = np.linspace(0.5, 0.3, T)[:, None]              # strictly improving (steps 0.018 >> 1e-6)
    assert O.stopping_check(improving, patience=3)[0] is None   # -> continue through t = T
    # flat hard WPSL for `patience` iterations while L keeps decreasing -> stop at the patience-th flat step
    flat = np.r_[np.linspace(0.5, 0.4, 5), np.full(T - 5, 0.4)][:, None]
    L = np.linspace(1.0, 0.5, T)[:, None]
    stop, bi, bw = O.stopping_check(flat, patience=3, lhist=L)
    assert stop == 5 + 3 and bi[0] == 5 and bw[0] == 0.4
    # the same flat WPSL while L rises: no stop (the criterion needs "further reduction of L")
    assert O.stopping_check(flat, patience=3, lhist=L[::-1].copy())[0] is None
    # improvements below the 1e-6 tolerance do not reset the window ("by >= 1e-6")
    creep = np.r_[np.linspace(0.5, 0.4, 5), 0.4 - 1e-7 * np.arange(1, T - 4)][:, None]
    assert O.stopping_check(creep, patience=3)[0] == 8
    # two restarts: stop only when every restart has stalled (best snapshot per restart)
    two = np.c_[flat[:, 0], improving[:, 0]]
    stop, bi, bw = O.stopping_check(two, patience=3)
    assert stop is None and bi[1] == T and bw[1] == improving[-1, 0]
    # best-snapshot monotonicity: the running best is nonincreasing
    rng = np.random.default_rng(3)
    h = rng.random((T, 2))
    prev = np.full(2, np.inf)
    for t in range(1, T + 1):
        _, _, b = O.stopping_check(h[:t], patience=0)
        assert (b <= prev).all()
        prev = b
