"""Chebyshev Doppler engine (include/sqngd.h SQNGD_ENGINE_CHEBYSHEV)
against the fp64 oracle, through the C-ABI, on the same seeded fp32 inputs.

The engine interpolates the AF in Doppler from Q exact node correlations; its error bound
(lr_tol = 1e-7 of ||s|| ||w|| = N) is far inside the parity bar, so the bar is the same as the
per-bin FFT engine's (tests/parity_util.py): |A| per cell 1e-4 rel + 1e-6 N, loss 1e-5 rel,
PSL 0.01 dB, argmax identical when unique by > 1e-5, gradients 1e-4 normwise and 1e-3 component-wise.  Every case forces
the engine, and both engines are also compared with each other on the same inputs."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import C1, Cfg  # noqa: E402

from parity_util import check_grad, check_map  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
CHEB = sqngd.ENGINE_CHEBYSHEV


def T(a, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV, dtype=dtype)


def random_inputs(c, seed):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=seed)
    s = np.exp(2j * np.pi * z.astype(np.float64)).astype(np.complex64)
    w = inputs.random_complex((c.R, c.M, c.N), seed + 100)
    w = (w * np.sqrt(c.N / np.sum(np.abs(w.astype(np.complex128)) ** 2, axis=-1, keepdims=True))).astype(np.complex64)
    return s, w


def weights_for(c, seed):
    """Seeded non-negative w(tau, f) with some zero cells (excluded from the ROI, Eqs. 8-9)."""
    rng = np.random.default_rng(seed)
    wt = rng.uniform(0.5, 1.5, size=(c.K, c.lags)).astype(np.float32)
    wt[rng.uniform(size=wt.shape) < 0.1] = 0.0
    return wt


def argmax_unique(v_sorted):
    return len(v_sorted) < 2 or v_sorted[0] - v_sorted[1] > 1e-5 * v_sorted[0]


def roi_values(A, c, auto, wts=None):
    v = np.abs(A) / c.N
    if wts is not None:
        v = v * wts[None, None, None]
    tau = np.arange(-(c.N - 1), c.N)
    roi = (tau >= c.tlo) & (tau <= c.thi)
    out = []
    for m in range(c.M):
        for l in range(c.M):
            if (m == l) != auto:
                continue
            mk = np.broadcast_to(roi, v.shape[-2:]).copy()
            if auto and c.exclude_auto_zero_delay:
                mk[:, c.N - 1] = False
            if wts is not None:
                mk &= wts > 0
            out.append(v[:, m, l][:, mk].ravel())
    return np.sort(np.concatenate(out))[::-1] if out else np.zeros(0)


def fwd_cases():
    return [
        C1,
        Cfg("ragged", M=3, N=37, B=8, K=15, f_lo=-0.5, f_hi=0.5, r_n=3),
        Cfg("batch", M=2, N=48, B=4, K=21, f_lo=-0.5, f_hi=0.5, R=3),
        Cfg("roi", M=2, N=40, B=4, K=31, f_lo=-0.5, f_hi=0.5, tau_lo=-10, tau_hi=25),
        Cfg("offcentre", M=2, N=100, B=4, K=40, f_lo=0.2, f_hi=1.1),         # even K, shifted grid
        Cfg("wide", M=2, N=64, B=4, K=61, f_lo=-1.5, f_hi=1.5),              # more nodes
        Cfg("p2048", M=2, N=1024, B=16, K=33, f_lo=-0.5, f_hi=0.5),
        Cfg("p8192", M=2, N=4096, B=16, K=33, f_lo=-0.5, f_hi=0.5),       # cross maps at P = 8192
        Cfg("n2", M=2, N=2, B=2, K=31, f_lo=-0.5, f_hi=0.5, r_n=1),          # 3 lags, one 16-lag chunk
        Cfg("m1", M=1, N=33, B=4, K=63, f_lo=-0.5, f_hi=0.5),                 # no cross maps
        Cfg("k3", M=2, N=40, B=4, K=3, f_lo=-0.05, f_hi=0.05),               # one bin pair + middle, Q = 6
        Cfg("k5", M=2, N=40, B=4, K=5, f_lo=-0.5, f_hi=0.5),                 # partial tile, Q = 10
    ]


@pytest.mark.parametrize("c", fwd_cases(), ids=lambda c: c.name)
@pytest.mark.parametrize("mode", [sqngd.LOSS_MAX, sqngd.LOSS_LSE, sqngd.LOSS_PNORM])
def test_forward_map_and_metrics(c, mode):
    c = c.with_(loss_mode=mode, beta_or_p={0: 0.0, 1: 200.0, 2: 16.0}[mode], doppler_engine=CHEB)
    s, w = random_inputs(c, 7)
    ctx = sqngd.Context(c)
    info = ctx.engine_info()
    assert info["engine"] == "chebyshev" and 4 <= info["Q"] <= 16 and info["err_bound"] <= 1e-7
    met_buf, p, amap = ctx.af_forward(T(s), T(w), want_map=True)
    ctx.sync()
    mg = ctx.metrics(met_buf)
    ref_met, ref_p, A = O.af(c, s, w, want_A=True)
    check_map(amap.cpu().numpy(), A, c.N)
    for r in range(c.R):
        g, o = mg[r], ref_met[r]
        for key in ("wapsl", "wcpsl", "wpsl"):
            if o[key] > 0:
                assert abs(20 * math.log10(g[key] / o[key])) < 0.01, (key, g[key], o[key])
        assert abs(g["loss"] - o["loss"]) <= 1e-5 * abs(o["loss"]), (g["loss"], o["loss"])
        assert g["n_cells"] == o["n_cells"]
        if argmax_unique(roi_values(A[r:r + 1], c, True)):
            assert g["argmax_auto"] == o["argmax_auto"]
        if c.M > 1 and argmax_unique(roi_values(A[r:r + 1], c, False)):
            assert g["argmax_cross"] == o["argmax_cross"]
        np.testing.assert_allclose(p.cpu().numpy()[r], ref_p[r], rtol=1e-6, atol=1e-7)


def grad_cases():
    return [
        Cfg("g-c1", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5, eps_w=0.4),
        Cfg("g-ragged", M=3, N=29, B=8, K=17, f_lo=-0.5, f_hi=0.5, r_n=3),
        Cfg("g-batch", M=2, N=256, B=8, K=32, f_lo=-0.5, f_hi=0.5, R=2),
        Cfg("g-p2048", M=2, N=1024, B=16, K=65, f_lo=-0.5, f_hi=0.5),
    ]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("c", grad_cases(), ids=lambda c: c.name)
@pytest.mark.parametrize("mode", [sqngd.LOSS_MAX, sqngd.LOSS_LSE, sqngd.LOSS_PNORM])
def test_gradients_explicit_waveform(c, mode):
    c = c.with_(loss_mode=mode, beta_or_p={0: 0.0, 1: 60.0, 2: 8.0}[mode], doppler_engine=CHEB)
    s, w = random_inputs(c, 11)
    ref_met, gw_ref, gs_ref = O.loss_grad(c, s, w)
    ctx = sqngd.Context(c)
    assert ctx.engine_info()["engine"] == "chebyshev"
    met, gw = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_FILTERS)
    gw = gw.cpu().numpy()
    mA = ctx.metrics(met)
    met, gs = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_TRANSMIT)
    gs = gs.cpu().numpy()
    mB = ctx.metrics(met)
    ctx.sync()
    for r in range(c.R):
        assert abs(mA[r]["loss"] - ref_met[r]["loss"]) <= 1e-5 * ref_met[r]["loss"]
        assert abs(mB[r]["loss"] - ref_met[r]["loss"]) <= 1e-5 * ref_met[r]["loss"]
    check_grad(gw, gw_ref, "grad_w")
    check_grad(gs, gs_ref, "grad_s")


@pytest.mark.parametrize("engine", [sqngd.ENGINE_FFT, CHEB])
@pytest.mark.parametrize("mode", [sqngd.LOSS_LSE, sqngd.LOSS_PNORM])
def test_weighted_roi(engine, mode):
    """Weighted peak sidelobe (Eqs. 8-9 with w(tau, f)): map-free metrics and both gradients."""
    c = Cfg("w", M=2, N=48, B=4, K=25, f_lo=-0.5, f_hi=0.5, loss_mode=mode,
            beta_or_p={1: 60.0, 2: 8.0}[mode], doppler_engine=engine)
    s, w = random_inputs(c, 13)
    wt = weights_for(c, 5)
    ref_met, gw_ref, gs_ref = O.loss_grad(c, s, w, weights=wt)
    ctx = sqngd.Context(c, weights=wt)
    met, gw = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_FILTERS)
    mA = ctx.metrics(met)
    met, gs = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_TRANSMIT)
    mB = ctx.metrics(met)
    ctx.sync()
    o = ref_met[0]
    for g in (mA[0], mB[0]):
        assert abs(g["loss"] - o["loss"]) <= 1e-5 * o["loss"]
        assert abs(20 * math.log10(g["wpsl"] / o["wpsl"])) < 0.01
        assert g["n_cells"] == o["n_cells"]
    check_grad(gw.cpu().numpy(), gw_ref, "grad_w (weighted)")
    check_grad(gs.cpu().numpy(), gs_ref, "grad_s (weighted)")


def test_engines_agree_and_ksplit():
    """Both engines on the same C2-shaped inputs (a k-split of the Chebyshev units): maps within
    the parity bar of each other, gradients within 1e-4."""
    c = Cfg("c2ish", M=4, N=256, B=8, K=129, f_lo=-0.5, f_hi=0.5, loss_mode=sqngd.LOSS_LSE, beta_or_p=200.0)
    s, w = random_inputs(c, 17)
    out = {}
    for eng in (sqngd.ENGINE_FFT, CHEB):
        ctx = sqngd.Context(c.with_(doppler_engine=eng))
        met, p, amap = ctx.af_forward(T(s), T(w), want_map=True)
        m1 = ctx.metrics(met)[0]
        _, gs = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_TRANSMIT)
        _, gw = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_FILTERS)
        ctx.sync()
        out[eng] = (amap.cpu().numpy().astype(np.float64), m1, gs.cpu().numpy(), gw.cpu().numpy())
    a0, m0, gs0, gw0 = out[sqngd.ENGINE_FFT]
    a1, m1, gs1, gw1 = out[CHEB]
    assert np.all(np.abs(a1 - a0) <= 1e-4 * a0 + 1e-6 * c.N)
    assert abs(m1["loss"] - m0["loss"]) <= 1e-5 * m0["loss"]
    assert rel(gs1, gs0) < 1e-4 and rel(gw1, gw0) < 1e-4


def test_transmit_chain_and_step():
    """The (z, rho) chain and one graph-replayed A+B block on the Chebyshev engine against the
    oracle (teacher-forced gradients and the hard-waveform metrics of the iterate the block starts from)."""
    c = Cfg("chain", M=2, N=48, B=4, K=31, f_lo=-0.5, f_hi=0.5, r_n=4, c=60.0, loss_mode=sqngd.LOSS_LSE,
            beta_or_p=60.0, doppler_engine=CHEB, n_h=2, n_x=2, lr_z=1e-3)
    z = inputs.phase_params(1, c.M, c.N, config_index=9)
    rho = inputs.random_sorted_thresholds(1, c.B, c.r_n, seed=4)
    _, w = random_inputs(c, 21)
    q = O.quantize(c, z, rho)
    _, _, gs = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs)
    ctx = sqngd.Context(c)
    _, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
    ctx.sync()
    assert rel(gz.cpu().numpy(), gz_ref) < 1e-4
    assert rel(gr.cpu().numpy(), gr_ref) < 1e-4
    st = ctx.new_state(T(z), T(rho), T(w))
    hard = torch.empty(sqngd.METRICS_BYTES, dtype=torch.uint8, device=DEV)
    hist = torch.zeros((1, 4), dtype=torch.float64, device=DEV)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
    side.synchronize()
    ctx.sync()
    h = hist.cpu().numpy()[0]
    assert np.isfinite(h).all() and (h > 0).all()
    # hard_out: the entry iterate (z, rho, w), scored by Step A's first evaluation; its loss is that
    # evaluation's (loss history column 0), its SNRL from the literal norms (Eq. 10)
    hm = sqngd.metrics_from_bytes(hard.cpu().numpy())[0]
    q2 = O.quantize(c, z, rho)
    om, _, _ = O.af(c, q2["s_hard"], w)
    assert abs(hm["wpsl"] - om[0]["wpsl"]) <= 1e-4 * om[0]["wpsl"]
    assert abs(hm["loss"] - om[0]["loss"]) <= 1e-5 * abs(om[0]["loss"])
    assert hm["loss"] == h[0]
    assert abs(hm["snrl_db_max"] - max(O.snrl_db(q2["s_hard"][0, m], w[0, m]) for m in range(c.M))) <= 1e-6


def test_engine_selection():
    """AUTO picks Chebyshev on the paper's narrow grid (Q = 10 for the 1e-7 bound), the FFT engine
    on C4's full-band grid; forcing Chebyshev where Q > 16 would be needed is rejected."""
    for name, eng, q in [("C1", "chebyshev", 10), ("C3", "chebyshev", 10)]:
        from paper_2604_25728_b200.configs import CONFIGS
        ctx = sqngd.Context(CONFIGS[name])
        info = ctx.engine_info()
        assert info["engine"] == eng and info["Q"] == q, info
        ctx.close()
    from paper_2604_25728_b200.configs import C4
    assert sqngd.Context(C4).engine_info()["engine"] == "fft"
    with pytest.raises(sqngd.SqngdError):
        sqngd.Context(C4.with_(doppler_engine=CHEB))


def test_step_A_teacher_forced():
    """One Step-A inner step on the Chebyshev engine (R = 2, R M = 6 rows): Adam(Re w, Im w) + Pi_H
    applied to the GPU's own grad_w equals the oracle's."""
    c = Cfg("stepA", M=3, N=40, B=4, K=31, f_lo=-0.5, f_hi=0.5, r_n=4, R=2, loss_mode=sqngd.LOSS_LSE,
            beta_or_p=60.0, doppler_engine=CHEB, n_h=1, n_x=1, lr_w=5e-2)
    z = inputs.phase_params(c.R, c.M, c.N, config_index=19)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z), T(rho), T(w))
    _, gw = ctx.af_loss_grad(st["z"], st["rho"], st["w"], sqngd.WRT_FILTERS)
    ctx.sync()
    gw = gw.cpu().numpy().astype(np.complex128)
    q = O.quantize(c, z, rho)
    _, gw_ref, _ = O.loss_grad(c, q["s_hard"], w, want_w=True, want_s=False)
    assert rel(gw, gw_ref) < 1e-4
    ctx.step(st, sqngd.BLOCK_A)
    ctx.sync()
    ost = O.new_state(z, rho, w)
    O.step(c, ost, block=1, grads_from=lambda kind, i, s_: gw)
    np.testing.assert_allclose(st["w"].cpu().numpy(), ost["w"], rtol=0, atol=2e-6)
