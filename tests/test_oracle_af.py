"""Pins of the oracle's AF/CAF and metrics against things other than itself:
numpy.correlate, closed forms (Dirichlet kernel, Parseval volume, sum over lags),
symmetry, Barker-13, and the SPEC worked examples (tests/golden)."""
import math
import os
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def cfg(M=1, N=8, K=1, f_lo=0.0, f_hi=0.0, R=1, **kw):
    d = dict(R=R, M=M, N=N, B=4, r_n=1, c=300.0, K=K, f_lo=f_lo, f_hi=f_hi, tau_lo=None, tau_hi=None,
             exclude_auto_zero_delay=1, loss_mode=0, beta_or_p=0.0, eps_w=0.1, mu_db=0.5)
    d.update(kw)
    return SimpleNamespace(**d)


def rnd(shape, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


def golden_values(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        if line.startswith("#") or not line.strip():
            continue
        k, v = line.split()
        out[k] = float(v)
    return out


@pytest.mark.parametrize("N", [1, 2, 5, 16, 33])
def test_zero_doppler_equals_numpy_correlate(N):
    s = rnd((1, 1, N), 1 + N)
    w = rnd((1, 1, N), 100 + N)
    _, _, A = O.af(cfg(N=N), s, w, want_A=True)
    ref = np.conj(np.correlate(w[0, 0], s[0, 0], mode="full"))  # index tau + N - 1
    np.testing.assert_allclose(A[0, 0, 0, 0], ref, rtol=0, atol=1e-12 * N)


@pytest.mark.parametrize("N,K,flo,fhi", [(8, 9, -3.0, 3.0), (13, 7, -0.5, 0.5), (32, 5, -16.0, 16.0)])
def test_dirichlet_closed_form(N, K, flo, fhi):
    """s = w = 1: |A(tau,f)| = |sin(pi f (N-|tau|)/N) / sin(pi f / N)| (N - |tau| when f/N is an integer)."""
    c = cfg(N=N, K=K, f_lo=flo, f_hi=fhi)
    one = np.ones((1, 1, N), complex)
    _, _, A = O.af(c, one, one, want_A=True)
    fk = O.doppler_grid(c)
    for k, f in enumerate(fk):
        for tau in range(-(N - 1), N):
            L = N - abs(tau)
            if abs(math.sin(math.pi * f / N)) < 1e-15:
                ref = L
            else:
                ref = abs(math.sin(math.pi * f * L / N) / math.sin(math.pi * f / N))
            assert abs(abs(A[0, 0, 0, k, tau + N - 1]) - ref) < 1e-12 * N


@pytest.mark.parametrize("N", [4, 9, 16])
def test_parseval_volume_on_integer_grid(N):
    """sum_{tau, f=0..N-1} |A|^2 = N ||s||^2 ||w||^2 (DFT over n of the lag product)."""
    c = cfg(M=2, N=N, K=N, f_lo=0.0, f_hi=float(N - 1))
    s = rnd((1, 2, N), 7)
    w = rnd((1, 2, N), 8)
    _, _, A = O.af(c, s, w, want_A=True)
    for m in range(2):
        for l in range(2):
            vol = np.sum(np.abs(A[0, m, l]) ** 2)
            ref = N * np.sum(np.abs(s[0, m]) ** 2) * np.sum(np.abs(w[0, l]) ** 2)
            assert abs(vol - ref) < 1e-10 * ref


def test_sum_over_lags_factorizes():
    """sum_tau A(tau, f) = (sum_n s(n) e^{j2pi n f/N}) * conj(sum_k w(k))."""
    N, K = 11, 5
    c = cfg(M=1, N=N, K=K, f_lo=-2.0, f_hi=2.0)
    s, w = rnd((1, 1, N), 3), rnd((1, 1, N), 4)
    _, _, A = O.af(c, s, w, want_A=True)
    n = np.arange(1, N + 1)
    for k, f in enumerate(O.doppler_grid(c)):
        lhs = A[0, 0, 0, k].sum()
        rhs = np.sum(s[0, 0] * np.exp(2j * np.pi * n * f / N)) * np.conj(np.sum(w[0, 0]))
        assert abs(lhs - rhs) < 1e-11 * N * N


def test_auto_symmetry():
    """w = s: |A(-tau, -f)| = |A(tau, f)| on a symmetric grid."""
    N, K = 12, 7
    c = cfg(M=1, N=N, K=K, f_lo=-0.75, f_hi=0.75)
    s = rnd((1, 1, N), 5)
    _, _, A = O.af(c, s, s, want_A=True)
    a = np.abs(A[0, 0, 0])
    np.testing.assert_allclose(a, a[::-1, ::-1], atol=1e-12 * N)


def test_zero_zero_is_inner_product_and_cauchy_schwarz():
    N = 10
    c = cfg(M=2, N=N, K=3, f_lo=-0.5, f_hi=0.5)
    s, w = rnd((1, 2, N), 9), rnd((1, 2, N), 10)
    met, p, A = O.af(c, s, w, want_A=True)
    for m in range(2):
        ip = np.sum(s[0, m] * np.conj(w[0, m]))
        assert abs(A[0, m, m, 1, N - 1] - ip) < 1e-12 * N
        assert abs(p[0, m] - abs(ip) / N) < 1e-14
        bound = np.linalg.norm(s[0, m]) * np.linalg.norm(w[0, :], axis=1).max()
        assert np.abs(A[0, m]).max() <= bound * (1 + 1e-12)


def test_spec_examples():
    one4 = np.ones((1, 1, 4), complex)
    c = cfg(N=4, K=3, f_lo=0.0, f_hi=2.0)   # f in {0, 1, 2}
    _, _, A = O.af(c, one4, one4, want_A=True)
    assert abs(A[0, 0, 0, 0, 3] - 4) < 1e-12        # A(0,0) = 4
    assert abs(A[0, 0, 0, 0, 6] - 1) < 1e-12        # A(3,0) = 1
    assert abs(A[0, 0, 0, 2, 3]) < 1e-12            # A(0,f=2) = 0
    # Doppler modulation x = 1, N = 4, f = 2 -> [-1, 1, -1, 1]: read it through impulse filters.
    xhat = []
    for n in range(4):
        e = np.zeros((1, 1, 4), complex)
        e[0, 0, n] = 1.0
        _, _, A = O.af(cfg(N=4, K=1, f_lo=2.0, f_hi=2.0), one4, e, want_A=True)
        xhat.append(A[0, 0, 0, 0, 3])
    np.testing.assert_allclose(xhat, [-1, 1, -1, 1], atol=1e-12)
    # [1,1] autocorrelation -> (1, 2, 1)
    two = np.ones((1, 1, 2), complex)
    _, _, A = O.af(cfg(N=2), two, two, want_A=True)
    np.testing.assert_allclose(A[0, 0, 0, 0], [1, 2, 1], atol=1e-12)
    # all-ones N=4 matched: WAPSL = 3/4 (tau = 0 column excluded, /N)
    met, _, _ = O.af(cfg(N=4), one4, one4)
    assert abs(met[0]["wapsl"] - 0.75) < 1e-14
    assert met[0]["flags"] & 1 and met[0]["wcpsl"] == 0.0   # M = 1: no cross terms


def test_barker13_pslr():
    lines = [l for l in open(os.path.join(GOLD, "barker13.txt")) if not l.startswith("#")]
    code = np.array([float(x) for x in lines[0].split()])
    want_db = float(lines[1])
    s = code.reshape(1, 1, 13).astype(complex)
    met, _, A = O.af(cfg(N=13), s, s, want_A=True)
    assert abs(met[0]["wapsl"] - 1.0 / 13) < 1e-14
    assert round(20 * math.log10(met[0]["wapsl"]), 2) == want_db
    side = np.abs(A[0, 0, 0, 0]).copy()
    side[12] = 0
    assert abs(side.max() - 1.0) < 1e-12


def test_tie_flag_barker13_and_constructions():
    """Flag 2 (SQNGD_FLAG_TIE): the maximum is attained by more than one cell.
    Barker-13 at zero Doppler has its 12 unit sidelobes exactly tied (integer sums, exact in fp64);
    two identical channels tie their auto maps (and their cross maps); a generic random pair does not."""
    lines = [l for l in open(os.path.join(GOLD, "barker13.txt")) if not l.startswith("#")]
    code = np.array([float(x) for x in lines[0].split()]).reshape(1, 1, 13).astype(complex)
    met, _, _ = O.af(cfg(N=13), code, code)
    assert met[0]["flags"] & 2
    s1 = np.exp(2j * np.pi * np.random.default_rng(5).random(40))
    w1 = s1 * np.exp(0.3j * np.arange(40) ** 0.5)
    s = np.stack([s1, s1])[None]
    w = np.stack([w1, w1])[None]
    met, _, _ = O.af(cfg(M=2, N=40, K=7, f_lo=-0.5, f_hi=0.5), s, w)
    assert met[0]["flags"] & 2 and met[0]["argmax_auto"][:2] == (0, 0)
    # (mismatched: with w = s the auto maps' |A(-tau, -f)| = |A(tau, f)| symmetry ties them too)
    met, _, _ = O.af(cfg(M=2, N=40, K=7, f_lo=-0.5, f_hi=0.5), rnd((1, 2, 40), 91), rnd((1, 2, 40), 93))
    assert not met[0]["flags"] & 2
    met, _, _ = O.af(cfg(M=2, N=40, K=7, f_lo=-0.5, f_hi=0.5), s, s.copy())
    assert met[0]["flags"] & 2
    # one tied pair planted by symmetry: a real code's |A(tau, -f)| = |A(tau, f)|, and the grid is symmetric
    x = np.sign(rnd((1, 1, 31), 92).real).astype(complex)
    met, _, A = O.af(cfg(N=31, K=5, f_lo=-0.5, f_hi=0.5, exclude_auto_zero_delay=1), x, x, want_A=True)
    v = np.abs(A[0, 0, 0]).copy()
    v[:, 30] = -1
    n_max = int(np.sum(v == v.max()))
    assert n_max >= 2 and bool(met[0]["flags"] & 2) == (n_max >= 2)


def test_snrl_and_targets():
    g = golden_values("spec_examples.txt")
    # Eq. 10 via p_m: SNRL = 10 log10(||x||^2 ||h||^2 / (N p)^2)
    x = np.array([[[1, 1]]], complex)
    h = np.array([[[1, 0]]], complex)
    _, p, _ = O.af(cfg(N=2), x, h)
    snrl = 10 * math.log10(np.sum(abs(x) ** 2) * np.sum(abs(h) ** 2) / (2 * p[0, 0]) ** 2)
    assert abs(snrl - g["snrl_db_example"]) < 1e-4
    # p_tar through the loss: eps = 0, matched (p = 1) -> L = (1 - p_tar)^2
    for mu, key in ((0.5, "p_tar_0p5"), (6.0206, "p_tar_6p0206")):
        s = np.exp(2j * np.pi * np.random.default_rng(1).random((1, 2, 8)))
        met, _, _ = O.af(cfg(M=2, N=8, eps_w=0.0, mu_db=mu), s, s)
        ptar = 1 - math.sqrt(met[0]["loss_snrl"])
        assert abs(ptar - g[key]) < 5e-6
        assert abs(met[0]["loss"] - met[0]["loss_snrl"]) < 1e-15


def test_eps_endpoint_and_max_tie_order():
    N = 9
    s, w = rnd((1, 2, N), 11), rnd((1, 2, N), 12)
    met, _, _ = O.af(cfg(M=2, N=N, K=3, f_lo=-1, f_hi=1, eps_w=1.0), s, w)
    m = met[0]
    assert m["loss"] == m["loss_wpsl"] == m["wpsl"] == max(m["wapsl"], m["wcpsl"])
    # A map with exact ties: s = w = 1 has |A(tau)| = |A(-tau)|; lowest (m,l,tau,k) must win.
    one = np.ones((1, 1, 6), complex)
    met, _, _ = O.af(cfg(N=6), one, one)
    assert met[0]["argmax_auto"] == (0, 0, -1, 0)


@pytest.mark.parametrize("mode,param", [(1, 4000.0), (2, 400.0)])
def test_surrogates_tend_to_max(mode, param):
    N = 10
    s, w = rnd((1, 2, N), 21), rnd((1, 2, N), 22)
    c = cfg(M=2, N=N, K=5, f_lo=-1, f_hi=1, loss_mode=mode, beta_or_p=param)
    met, _, _ = O.af(c, s, w)
    m = met[0]
    assert m["loss_wpsl"] >= m["wpsl"] * (1 - 1e-12)
    # LSE: wpsl <= L <= wpsl + ln|S|/beta ; PNORM: wpsl <= L <= |S|^{1/p} wpsl
    ub = m["wpsl"] + math.log(m["n_cells"]) / param if mode == 1 else m["wpsl"] * m["n_cells"] ** (1 / param)
    assert m["loss_wpsl"] <= ub * (1 + 1e-12)
    assert abs(m["loss_wpsl"] - m["wpsl"]) < 0.02 * m["wpsl"]


def test_roi_weights_and_lag_window():
    """Weights restrict the search: zero outside tau = +-1 -> 3/4 for all-ones N=4."""
    N, K = 4, 1
    wts = np.zeros((K, 2 * N - 1))
    wts[0, N - 2] = wts[0, N] = 1.0
    one = np.ones((1, 1, N), complex)
    met, _, _ = O.af(cfg(N=N), one, one, weights=wts)
    assert abs(met[0]["wapsl"] - 0.75) < 1e-14
    met, _, _ = O.af(cfg(N=N, tau_lo=2, tau_hi=3), one, one)
    assert abs(met[0]["wapsl"] - 0.5) < 1e-14


def test_snrl_db_pins():
    """O.snrl_db (Eq. 10) against SPEC's worked examples (h = x -> 0 dB,
    h = 2x -> 0 dB, N = 2 x = [1,1] h = [1,0] -> 10 log10 2), Cauchy-Schwarz (>= 0, = 0 only for
    h parallel to x) and the unimodular identity SNRL = -20 log10 p_m when ||x||^2 = ||h||^2 = N."""
    g = golden_values("spec_examples.txt")
    x = rnd(16, 3)
    assert abs(O.snrl_db(x, x)) < 1e-12
    assert abs(O.snrl_db(x, 2 * x)) < 1e-12
    assert abs(O.snrl_db(x, (0.5 - 2j) * x)) < 1e-12
    assert abs(O.snrl_db([1, 1], [1, 0]) - g["snrl_db_example"]) < 1e-4
    for seed in range(5):
        assert O.snrl_db(rnd(16, 10 + seed), rnd(16, 20 + seed)) > 0.0
    assert O.snrl_db([1, 0], [0, 1]) == float("inf")
    N = 32
    s = np.exp(2j * np.pi * np.random.default_rng(4).random((1, 1, N)))
    h = rnd((1, 1, N), 5)
    h *= math.sqrt(N) / np.linalg.norm(h)
    _, p, _ = O.af(cfg(N=N), s, h)
    assert abs(O.snrl_db(s, h) + 20 * math.log10(p[0, 0])) < 1e-10
