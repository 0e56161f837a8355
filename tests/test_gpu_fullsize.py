"""Parity at BASELINE.json's full sizes, in the configuration bench.py times (LSE, beta = 200,
matched start w = s_hard, seeds 1000*config + restart).  Where the oracle can afford it the
whole output is compared (C3 / C4 gradients, C4 map); otherwise sampled (m, l, k) rows of
the AF are recomputed by the oracle one by one, the reported maxima are checked at their
argmax cells, and properties that hold at any size are checked (C5)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402

from parity_util import check_grad, check_map, record  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda"


def T(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


ENGINES = {"fft": sqngd.ENGINE_FFT, "cheb": sqngd.ENGINE_CHEBYSHEV}


def bench_cfg(name, engine="auto"):
    """The bench configuration; `engine` forces a Doppler engine (auto: the library's choice,
    Chebyshev on the narrow grids C1-C3, C5; FFT on C4)."""
    c = CF.CONFIGS[name]
    return c.with_(loss_mode=CF.LOSS_LSE, beta_or_p=200.0, doppler_engine=ENGINES.get(engine, 0))


def bench_inputs(c):
    z = np.stack([inputs.uniform01_f32(inputs.config_seed(c.index, r), c.M * c.N).reshape(c.M, c.N)
                  for r in range(c.R)])
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    return z, rho


def oracle_row(c, s, w, r, m, l, k):
    """|A_ml(., f_k)| over all 2N-1 lags by the oracle (one pair, one bin)."""
    f = O.doppler_grid(c)[k]
    cc = c.with_(R=1, M=1, K=1, f_lo=float(f), f_hi=float(f))
    _, _, A = O.af(cc, s[r:r + 1, m:m + 1], w[r:r + 1, l:l + 1], want_A=True)
    return np.abs(A[0, 0, 0, 0])


def roi_mask(c, auto):
    tau = np.arange(-(c.N - 1), c.N)
    mk = (tau >= c.tlo) & (tau <= c.thi)
    if auto and c.exclude_auto_zero_delay:
        mk &= tau != 0
    return mk


def check_forward(c, want_map, rows):
    z, rho = bench_inputs(c)
    q = O.quantize(c, z, rho)
    ctx = sqngd.Context(c)
    out = ctx.quantize(T(z), T(rho))
    assert np.array_equal(out["b_hard"].cpu().numpy().astype(np.int32), q["b_hard"])
    s = out["s_hard"]
    w = s.clone()                                    # matched start (Q3)
    met, p, amap = ctx.af_forward(s, w, want_map=want_map)
    ctx.sync()
    mg = ctx.metrics(met)
    s64 = q["s_hard"]
    w64 = out["s_hard"].cpu().numpy().astype(np.complex128)
    np.testing.assert_allclose(s64, w64, atol=1e-7)
    g = np.random.default_rng(3)
    for _ in range(rows):
        r, m, l, k = g.integers(c.R), g.integers(c.M), g.integers(c.M), g.integers(c.K)
        ref = oracle_row(c, s64, w64, r, m, l, k)
        if amap is not None:
            got = amap[r, m, l, k].cpu().numpy().astype(np.float64)
            check_map(got, ref, c.N, what=f"{c.name} sampled row")
        vmax = ref[roi_mask(c, m == l)].max() / c.N
        assert vmax <= mg[r]["wpsl"] * (1 + 1e-4) + 1e-6
    for r in range(c.R):
        for key, arg in (("wapsl", "argmax_auto"), ("wcpsl", "argmax_cross")):
            m, l, tau, k = mg[r][arg]
            ref = oracle_row(c, s64, w64, r, m, l, k)[tau + c.N - 1] / c.N
            assert abs(mg[r][key] - ref) <= 1e-4 * ref + 1e-6, (key, mg[r][key], ref)
        lse = mg[r]["loss_wpsl"]
        assert mg[r]["wpsl"] * (1 - 1e-6) <= lse <= mg[r]["wpsl"] + math.log(mg[r]["n_cells"]) / 200.0 + 1e-6
        np.testing.assert_allclose(p.cpu().numpy()[r], 1.0, atol=1e-6)   # |<s, s>| / N = 1 at the matched start
    return ctx, mg


@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_c3_forward_sampled_rows_and_argmax(engine):
    check_forward(bench_cfg("C3", engine), want_map=True, rows=24)


def test_c4_forward_full_map():
    c = bench_cfg("C4")
    z, rho = bench_inputs(c)
    q = O.quantize(c, z, rho)
    s = q["s_hard"].astype(np.complex64)
    ctx = sqngd.Context(c)
    met, _, amap = ctx.af_forward(T(s), T(s), want_map=True)
    ctx.sync()
    ref_met, _, A = O.af(c, s, s, want_A=True)
    ref = np.abs(A)
    got = amap.cpu().numpy().astype(np.float64)
    check_map(got, ref, c.N, what="C4 full map")
    mg = ctx.metrics(met)[0]
    assert abs(mg["loss"] - ref_met[0]["loss"]) <= 1e-5 * ref_met[0]["loss"]
    assert abs(20 * math.log10(mg["wpsl"] / ref_met[0]["wpsl"])) < 0.01


@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_c5_forward_sampled_rows_and_argmax(engine):
    check_forward(bench_cfg("C5", engine), want_map=False, rows=12)


@pytest.mark.parametrize("name,engine", [("C3", "fft"), ("C3", "cheb"), ("C4", "fft")])
def test_full_gradients_vs_oracle(name, engine):
    """Step A (grad_w on s_hard) and Step B (grad_z, grad_rho through Q_A) against the full
    fp64 oracle at the benchmark size, with a perturbed (non-matched) filter bank."""
    c = bench_cfg(name, engine)
    z, rho = bench_inputs(c)
    q = O.quantize(c, z, rho)
    w = (q["s_hard"] * np.exp(0.3j * np.cos(np.arange(c.N)))).astype(np.complex64)
    ctx = sqngd.Context(c)
    met, gw = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_FILTERS)
    gw = gw.cpu().numpy()
    mA = ctx.metrics(met)[0]
    met, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
    gz, gr = gz.cpu().numpy(), gr.cpu().numpy()
    mB = ctx.metrics(met)[0]
    ctx.sync()
    refA, gw_ref, _ = O.loss_grad(c, q["s_hard"], w, want_s=False)
    refB, _, gs_ref = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs_ref)

    def rel(a, b):
        return np.linalg.norm(a - b) / np.linalg.norm(b)

    assert abs(mA["loss"] - refA[0]["loss"]) <= 1e-5 * refA[0]["loss"]
    assert abs(mB["loss"] - refB[0]["loss"]) <= 1e-5 * refB[0]["loss"]
    check_grad(gw, gw_ref, f"{name} grad_w")
    check_grad(gz, gz_ref, f"{name} grad_z")
    check_grad(gr, gr_ref, f"{name} grad_rho")


@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_c5_gradient_doppler_split_consistency(engine):
    """A property that holds at any size: the Step-B gradient of the full Doppler grid equals
    the max-then-sum combination (parallel.combine_lse arithmetic) of the gradients of its two
    halves, each evaluated by the same kernels (restart 0 of C5, P = 8192)."""
    c = bench_cfg("C5", engine).with_(R=1, eps_w=1.0)
    z, rho = bench_inputs(c.with_(R=1))
    q = O.quantize(c, z, rho)
    s = T(q["s_soft"].astype(np.complex64))
    w = T(q["s_hard"].astype(np.complex64))
    full = sqngd.Context(c)
    mf, gf = full.loss_grad_s(s, w, sqngd.WRT_TRANSMIT)
    gf = gf.cpu().numpy().astype(np.complex128)
    Lf = full.metrics(mf)[0]["loss_wpsl"]
    d = (c.f_hi - c.f_lo) / (c.K - 1)
    parts = []
    for k0, k1 in ((0, c.K // 2), (c.K // 2, c.K)):
        ch = c.with_(K=k1 - k0, f_lo=c.f_lo + k0 * d, f_hi=c.f_lo + (k1 - 1) * d)
        ctx = sqngd.Context(ch)
        mh, gh = ctx.loss_grad_s(s, w, sqngd.WRT_TRANSMIT)
        md = ctx.metrics(mh)[0]
        S = math.exp(200.0 * (md["loss_wpsl"] - md["wpsl"]))
        parts.append((md["wpsl"], S, gh.cpu().numpy().astype(np.complex128) * S))
        ctx.sync()
    m = max(p[0] for p in parts)
    S = sum(p[1] * math.exp(200.0 * (p[0] - m)) for p in parts)
    G = sum(p[2] * math.exp(200.0 * (p[0] - m)) for p in parts) / S
    assert abs((m + math.log(S) / 200.0) - Lf) <= 2e-6 * Lf
    assert np.linalg.norm(G - gf) / np.linalg.norm(gf) < 1e-4
