"""Shared parity checks of the GPU path (C-ABI) against the fp64 oracle, with a record of the
error each check actually achieved (DESIGN.md §4 "Parity bar").

Bars (SURVEY.md §8(c) "What pins each part", BASELINE north star):
  |A| per cell:  | |A|_gpu - |A|_ref | <= 1e-4 |A|_ref + 1e-6 N   (BASELINE "1e-4 relative" with the
                 survey's -60 dB absolute floor, 1e-6 N)
  gradients:     ||g_gpu - g_ref|| / ||g_ref|| <= 1e-4, and component-wise
                 |g_gpu - g_ref| <= 1e-3 |g_ref| wherever |g_ref| >= 1e-3 max |g_ref|
  loss:          1e-5 relative;  PSL: 0.01 dB;  s_soft phase: 1e-6 rad.

Every check appends (test id, quantity, achieved, bar) to RECORD; tests/conftest.py writes the
record to $SQNGD_PARITY_LOG at the end of the session (profiles/ keeps the GPU run's copy).
"""
from __future__ import annotations

import os

import numpy as np

MAP_REL = 1e-4
MAP_FLOOR = 1e-6          # x N
GRAD_NORM = 1e-4
GRAD_COMP = 1e-3
GRAD_COMP_SUPPORT = 1e-3  # components with |g_ref| >= this x max |g_ref|
LOSS_REL = 1e-5
PSL_DB = 0.01

RECORD: list[dict] = []


def _test_id() -> str:
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def record(quantity: str, achieved: float, bar: float, **extra) -> None:
    RECORD.append({"test": _test_id(), "quantity": quantity, "achieved": float(achieved), "bar": float(bar), **extra})


def check_map(A_gpu, A_ref, N, floor: float = MAP_FLOOR, what: str = "map") -> float:
    """Cell-by-cell |A| check; returns max |err| / N."""
    ref = np.abs(np.asarray(A_ref))
    err = np.abs(np.asarray(A_gpu, dtype=np.float64) - ref)
    excess = err - MAP_REL * ref
    worst = float(excess.max() / N) if excess.size else 0.0
    record(f"{what} max(|d|A|| - 1e-4|A|)/N", worst, floor)
    record(f"{what} max|d|A||/N", float(err.max() / N) if err.size else 0.0, floor + MAP_REL)
    bad = excess > floor * N
    assert not bad.any(), f"{bad.sum()} cells off; worst (|err| - 1e-4|ref|)/N = {worst:.3e} (floor {floor:g})"
    return worst


def rel(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def check_grad(g, g_ref, what: str = "grad") -> tuple[float, float]:
    """Normwise 1e-4 and component-wise 1e-3 on the support (>= 1e-3 of the largest component)."""
    g = np.asarray(g).astype(np.complex128 if np.iscomplexobj(g) else np.float64)
    g_ref = np.asarray(g_ref)
    nw = rel(g, g_ref)
    mag = np.abs(g_ref)
    sup = mag >= GRAD_COMP_SUPPORT * mag.max() if mag.size else mag.astype(bool)
    cw = float((np.abs(g - g_ref)[sup] / mag[sup]).max()) if sup.any() else 0.0
    record(f"{what} normwise", nw, GRAD_NORM)
    record(f"{what} componentwise", cw, GRAD_COMP, support=int(sup.sum()), size=int(mag.size))
    assert nw < GRAD_NORM, (what, "normwise", nw)
    assert cw <= GRAD_COMP, (what, "componentwise", cw, int(sup.sum()))
    return nw, cw


def check_loss(got: float, ref: float, what: str = "loss") -> float:
    r = abs(got - ref) / abs(ref)
    record(f"{what} rel", r, LOSS_REL)
    assert r <= LOSS_REL, (what, got, ref)
    return r


def check_db(got: float, ref: float, what: str = "psl") -> float:
    d = abs(20 * np.log10(got / ref))
    record(f"{what} dB", d, PSL_DB)
    assert d < PSL_DB, (what, got, ref)
    return d
