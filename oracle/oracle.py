"""ctypes wrapper of the fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  It never imports the CUDA package; configs are
duck-typed (any object with the attributes of the parameter block).

Functions mirror the hot path's semantics:
  quantize(cfg, z, rho)              O1  Eqs. 21-25, 43
  af(cfg, s, w, want_A)              O2/O3  Eqs. 6-10, 33-42
  loss_grad(cfg, s, w)               O4  closed-form adjoint sums
  chain(cfg, z, rho, s, grad_s)      O4  through Eqs. 23-24
  adam / project_filters / project_thresholds / step   O5 (Alg. 1)
  stopping_check(hist, patience, lhist)                 O6 (SPEC S:L542-550 stopping_check)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sqngd_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-shared", "-fPIC", "-Wall"]


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (separate from the CUDA build)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", *GCC_FLAGS, "-o", _LIB, _SRC])
    return _LIB


class OracleCfg(C.Structure):
    _fields_ = [
        ("R", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("B", C.c_int32), ("r_n", C.c_int32),
        ("c", C.c_double),
        ("K", C.c_int32),
        ("f_lo", C.c_double), ("f_hi", C.c_double),
        ("tau_lo", C.c_int32), ("tau_hi", C.c_int32),
        ("exclude_auto_zero_delay", C.c_int32),
        ("loss_mode", C.c_int32),
        ("beta_or_p", C.c_double),
        ("eps_w", C.c_double), ("mu_db", C.c_double),
        ("weights", C.POINTER(C.c_double)),
    ]


class OracleMetrics(C.Structure):
    _fields_ = [
        ("loss", C.c_double), ("loss_wpsl", C.c_double), ("loss_snrl", C.c_double),
        ("wapsl", C.c_double), ("wcpsl", C.c_double), ("wpsl", C.c_double),
        ("argmax_auto", C.c_int32 * 4), ("argmax_cross", C.c_int32 * 4),
        ("n_cells", C.c_int32), ("flags", C.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["argmax_auto"] = tuple(self.argmax_auto)
        d["argmax_cross"] = tuple(self.argmax_cross)
        return d


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        cp = C.POINTER(OracleCfg)
        _lib.oracle_QA.restype = C.c_double
        _lib.oracle_QA.argtypes = [C.c_int, C.c_int, C.c_double, dp, C.c_double]
        _lib.oracle_dQA.restype = C.c_double
        _lib.oracle_dQA.argtypes = [C.c_int, C.c_int, C.c_double, dp, C.c_double]
        _lib.oracle_QR_level.restype = C.c_int64
        _lib.oracle_QR_level.argtypes = [C.c_int, C.c_int, C.c_double, dp, C.c_double]
        _lib.oracle_quantize.argtypes = [cp, dp, dp, dp, dp, dp, ip, dp, dp]
        _lib.oracle_af.argtypes = [cp, dp, dp, dp, C.POINTER(OracleMetrics), dp]
        _lib.oracle_loss_grad.argtypes = [cp, dp, dp, C.POINTER(OracleMetrics), dp, dp]
        _lib.oracle_chain.argtypes = [cp, dp, dp, dp, dp, dp, dp]
        _lib.oracle_adam.argtypes = [C.c_int64, dp, dp, dp, dp, C.c_int64, C.c_double, C.c_double,
                                     C.c_double, C.c_double]
        _lib.oracle_project_filters.restype = C.c_int
        _lib.oracle_project_filters.argtypes = [C.c_int, C.c_int, dp]
        _lib.oracle_project_thresholds.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_double,
                                                   C.c_double]
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _c128(a):
    """complex -> interleaved fp64 (exact promotion of complex64)."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


class _Cfg:
    """Holds the ctypes block and keeps the weights buffer alive."""

    def __init__(self, cfg, R=None, weights=None):
        N = int(cfg.N)
        tlo = getattr(cfg, "tau_lo", None)
        thi = getattr(cfg, "tau_hi", None)
        self._w = None if weights is None else _f64(weights).reshape(int(cfg.K), 2 * N - 1)
        self.c = OracleCfg(
            R=int(cfg.R if R is None else R), M=int(cfg.M), N=N, B=int(cfg.B), r_n=int(cfg.r_n),
            c=float(cfg.c), K=int(cfg.K), f_lo=float(cfg.f_lo), f_hi=float(cfg.f_hi),
            tau_lo=-(N - 1) if tlo is None else int(tlo), tau_hi=(N - 1) if thi is None else int(thi),
            exclude_auto_zero_delay=int(getattr(cfg, "exclude_auto_zero_delay", 1)),
            loss_mode=int(getattr(cfg, "loss_mode", 0)), beta_or_p=float(getattr(cfg, "beta_or_p", 0.0)),
            eps_w=float(getattr(cfg, "eps_w", 0.1)), mu_db=float(getattr(cfg, "mu_db", 0.5)),
            weights=_dp(self._w),
        )

    def ref(self):
        return C.byref(self.c)


def doppler_grid(cfg) -> np.ndarray:
    K = int(cfg.K)
    if K == 1:
        return np.array([float(cfg.f_lo)])
    return float(cfg.f_lo) + (float(cfg.f_hi) - float(cfg.f_lo)) * np.arange(K) / (K - 1)


# ---------------------------------------------------------------- O1
def QA(B, r_n, c, rho, x) -> float:
    rho = _f64(rho)
    return lib().oracle_QA(B, r_n, c, _dp(rho), float(x))


def dQA(B, r_n, c, rho, x) -> float:
    rho = _f64(rho)
    return lib().oracle_dQA(B, r_n, c, _dp(rho), float(x))


def QR_level(B, r_n, c, rho, x) -> int:
    rho = _f64(rho)
    return int(lib().oracle_QR_level(B, r_n, c, _dp(rho), float(x)))


def quantize(cfg, z, rho, weights=None) -> dict:
    z = _f64(z)
    R = z.shape[0]
    rho = _f64(rho).reshape(R, -1)
    cc = _Cfg(cfg, R=R, weights=weights)
    shp = z.shape
    y_soft, dq, y_hard = np.empty(shp), np.empty(shp), np.empty(shp)
    b_hard = np.empty(shp, dtype=np.int32)
    s_soft, s_hard = np.empty(shp, np.complex128), np.empty(shp, np.complex128)
    lib().oracle_quantize(cc.ref(), _dp(z), _dp(rho), _dp(y_soft), _dp(dq), _dp(y_hard),
                          b_hard.ctypes.data_as(C.POINTER(C.c_int32)),
                          s_soft.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                          s_hard.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
    return dict(y_soft=y_soft, dq=dq, y_hard=y_hard, b_hard=b_hard, s_soft=s_soft, s_hard=s_hard)


# ---------------------------------------------------------------- O2/O3
def af(cfg, s, w, want_A: bool = False, weights=None):
    """Returns (metrics list[dict], p [R][M], A or None [R][M][M][K][2N-1])."""
    s, w = _c128(s), _c128(w)
    R = s.shape[0]
    cc = _Cfg(cfg, R=R, weights=weights)
    M, N, K = int(cfg.M), int(cfg.N), int(cfg.K)
    A = np.empty((R, M, M, K, 2 * N - 1), np.complex128) if want_A else None
    met = (OracleMetrics * R)()
    p = np.empty((R, M))
    lib().oracle_af(cc.ref(), _dp(s.view(np.float64)), _dp(w.view(np.float64)),
                    None if A is None else _dp(A.view(np.float64)), met, _dp(p))
    return [m.as_dict() for m in met], p, A


def snrl_db(x, h) -> float:
    """Eq. 10: SNRL = 10 log10(||x||^2 ||h||^2 / |x^H h|^2), the literal definition in fp64
    (+inf when x^H h = 0)."""
    x, h = _c128(x).ravel(), _c128(h).ravel()
    c = abs(np.vdot(x, h)) ** 2            # |x^H h|^2
    if c == 0.0:
        return float("inf")
    return float(10.0 * np.log10(np.vdot(x, x).real * np.vdot(h, h).real / c))


# ---------------------------------------------------------------- O4
def loss_grad(cfg, s, w, want_w: bool = True, want_s: bool = True, weights=None):
    """Returns (metrics list, grad_w = 2 dL/dw^*, grad_s = dL/ds^*)."""
    s, w = _c128(s), _c128(w)
    R = s.shape[0]
    cc = _Cfg(cfg, R=R, weights=weights)
    met = (OracleMetrics * R)()
    gw = np.zeros(s.shape, np.complex128) if want_w else None
    gs = np.zeros(s.shape, np.complex128) if want_s else None
    lib().oracle_loss_grad(cc.ref(), _dp(s.view(np.float64)), _dp(w.view(np.float64)), met,
                           None if gw is None else _dp(gw.view(np.float64)),
                           None if gs is None else _dp(gs.view(np.float64)))
    return [m.as_dict() for m in met], gw, gs


def chain(cfg, z, rho, s, grad_s):
    """dL/dz and dL/drho from g = dL/ds^* (Eqs. 23-24)."""
    z, s, grad_s = _f64(z), _c128(s), _c128(grad_s)
    R = z.shape[0]
    rho = _f64(rho).reshape(R, -1)
    cc = _Cfg(cfg, R=R)
    gz = np.empty(z.shape)
    gr = np.empty(rho.shape)
    lib().oracle_chain(cc.ref(), _dp(z), _dp(rho), _dp(s.view(np.float64)), _dp(grad_s.view(np.float64)),
                       _dp(gz), _dp(gr))
    return gz, gr


# ---------------------------------------------------------------- O5
def adam(x, m, v, g, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """In-place bias-corrected Adam on float64 arrays; t is the step number (>= 1)."""
    for a in (x, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = _f64(g)
    lib().oracle_adam(x.size, _dp(x), _dp(m), _dp(v), _dp(g), int(t), lr, b1, b2, eps)


def project_filters(w: np.ndarray) -> int:
    """In place on complex128 [..., N]; returns the number of zero rows."""
    assert w.dtype == np.complex128 and w.flags.c_contiguous
    N = w.shape[-1]
    return lib().oracle_project_filters(w.size // N, N, _dp(w.view(np.float64)))


def project_thresholds(rho: np.ndarray, lo=1e-4, hi=1 - 1e-4, gap=1e-6):
    assert rho.dtype == np.float64 and rho.flags.c_contiguous
    n = rho.shape[-1]
    lib().oracle_project_thresholds(rho.size // n, n, _dp(rho), lo, hi, gap)


def step(cfg, state: dict, block: int = 3, grads_from=None):
    """One Alg. 1 outer iteration on an fp64 state dict
    {z, rho, w, m_z, v_z, m_rho, v_rho, m_w, v_w, t_a, t_b} (modified in place).

    Step A (block & 1): n_h times [loss_grad on X_hard -> Adam(Re w, Im w) -> Pi_H].
    Step B (block & 2): n_x times [loss_grad on X_soft -> chain -> Adam(z), Adam(rho) -> rho projection].
    `grads_from`, if given, is a callable(kind, i, state) -> gradient arrays used
    instead of the oracle's own (teacher forcing of Adam with an external gradient); in
    generator mode Step B's pair is (dL/dtheta, dL/drho).
    Generator mode (state["theta"] set, NEXT-2): z = f_theta(y0) at the start and after every
    Step-B update; Step B's Adam acts on theta (rate cfg.lr_theta) instead of z (Alg. 1).
    Returns the per-inner-step loss history.
    """
    st = state
    hist = []
    net = st.get("theta") is not None  # generator mode (NEXT-2): z = f_theta(y0), Adam on theta
    if net:
        st["z"] = _net_z(cfg, st)
    if block & 1:
        q = quantize(cfg, st["z"], st["rho"])
        for i in range(int(cfg.n_h)):
            met, gw, _ = loss_grad(cfg, q["s_hard"], st["w"], want_w=True, want_s=False)
            if grads_from is not None:
                gw = grads_from("A", i, st)
            hist.append([m["loss"] for m in met])
            st["t_a"] += 1
            wv = st["w"].view(np.float64)
            adam(wv, st["m_w"], st["v_w"], np.ascontiguousarray(gw).view(np.float64), st["t_a"], cfg.lr_w,
                 cfg.adam_b1, cfg.adam_b2, cfg.adam_eps)
            project_filters(st["w"])
    if block & 2:
        for i in range(int(cfg.n_x)):
            q = quantize(cfg, st["z"], st["rho"])
            met, _, gs = loss_grad(cfg, q["s_soft"], st["w"], want_w=False, want_s=True)
            gz, gr = chain(cfg, st["z"], st["rho"], q["s_soft"], gs)
            if grads_from is not None:
                gz, gr = grads_from("B", i, st)
            hist.append([m["loss"] for m in met])
            st["t_b"] += 1
            if net:  # z = f_theta(y0): dL/dtheta through the generator (Eq. 20)
                if grads_from is None:
                    gth = _net_grad(cfg, st, gz)
                else:
                    gth = gz
                adam(st["theta"], st["m_theta"], st["v_theta"], gth, st["t_b"], cfg.lr_theta, cfg.adam_b1,
                     cfg.adam_b2, cfg.adam_eps)
            else:
                adam(st["z"], st["m_z"], st["v_z"], gz, st["t_b"], cfg.lr_z, cfg.adam_b1, cfg.adam_b2,
                     cfg.adam_eps)
            adam(st["rho"], st["m_rho"], st["v_rho"], gr, st["t_b"], cfg.lr_z, cfg.adam_b1, cfg.adam_b2,
                 cfg.adam_eps)
            project_thresholds(st["rho"])
            if net:
                st["z"] = _net_z(cfg, st)
    return np.array(hist)


def _net_dims(cfg):
    return int(cfg.M) * int(cfg.N), int(cfg.net_width), int(cfg.net_depth)


def _net_z(cfg, st):
    from oracle import net_oracle as NO

    Din, W, D = _net_dims(cfg)
    R = st["theta"].shape[0]
    z, st["_tapes"] = NO.forward_batch(st["theta"], st["y0"], Din, W, D)
    return np.ascontiguousarray(z.reshape(R, int(cfg.M), int(cfg.N)))


def _net_grad(cfg, st, gz):
    from oracle import net_oracle as NO

    Din, W, D = _net_dims(cfg)
    R = st["theta"].shape[0]
    return np.ascontiguousarray(NO.backward_batch(st["theta"], st["_tapes"], np.asarray(gz).reshape(R, Din), Din, W, D))


def new_state(z, rho, w, theta=None, y0=None) -> dict:
    """fp64 optimizer state; with theta [R][P] and y0 [R][M N] the generator parameterizes z
    (z is then recomputed as f_theta(y0) by step())."""
    z = _f64(z).copy()
    rho = _f64(rho).copy()
    w = _c128(w).copy()
    st = dict(z=z, rho=rho, w=w, m_z=np.zeros_like(z), v_z=np.zeros_like(z),
              m_rho=np.zeros_like(rho), v_rho=np.zeros_like(rho),
              m_w=np.zeros(w.size * 2), v_w=np.zeros(w.size * 2), t_a=0, t_b=0, theta=None)
    if theta is not None:
        st["theta"] = _f64(theta).copy()
        st["y0"] = _f64(y0).copy()
        st["m_theta"] = np.zeros_like(st["theta"])
        st["v_theta"] = np.zeros_like(st["theta"])
    return st


# ---------------------------------------------------------------- O6
def stopping_check(hist, patience, lhist=None, tol=1e-6):
    """Algorithm 1's stopping criterion over an outer-iteration history, as SPEC S:L542-545 reads
    P:L485 ("Training terminates when further reduction of L does not lead to improvement in the
    WPSL"): an improvement is a decrease of the best hard WPSL (linear, N-normalized) by more than
    `tol` = 1e-6; stop at the first outer iteration t (1-based) at which every restart has gone
    `patience` iterations without one while (lhist given) its loss L is below its value at its last
    improvement, i.e. L kept decreasing over the window.  (t = T stops Algorithm 1 regardless, P:L534;
    the caller's loop bound.)  hist, lhist: [T][R].  Returns (stop t or None, best_iter [R] (0: none),
    best_wpsl [R])."""
    hist = np.asarray(hist, dtype=np.float64)
    T, R = hist.shape
    best = np.full(R, np.inf)
    bi = np.zeros(R, int)
    stall = np.zeros(R, int)
    lref = np.zeros(R)
    for t in range(1, T + 1):
        for r in range(R):
            v = hist[t - 1, r]
            if v < best[r] - tol:
                best[r], bi[r], stall[r] = v, t, 0
                if lhist is not None:
                    lref[r] = lhist[t - 1, r]
            else:
                stall[r] += 1
        dec = np.ones(R, bool) if lhist is None else np.asarray(lhist)[t - 1] < lref
        if patience > 0 and ((stall >= patience) & dec).all():
            return t, bi, best
    return None, bi, best
