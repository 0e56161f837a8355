"""GPU (C-ABI) vs fp64 oracle on identical seeded fp32 inputs.

Tolerances (BASELINE north star):
  |A| per cell: | |A|_gpu - |A|_ref | <= 1e-4 |A|_ref + 1e-6 N      (tests/parity_util.py)
  loss:         relative 1e-5;   PSL: 0.01 dB;   argmax identical when unique by > 1e-5 rel.
  gradients:    ||g_gpu - g_ref|| / ||g_ref|| <= 1e-4, component-wise 1e-3 on the support
  hard phase indices: bit-exact.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import C1, Cfg  # noqa: E402

from parity_util import check_grad, check_map, record  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda"


def T(a, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV, dtype=dtype)


def cases_fwd():
    return [
        Cfg("tiny", M=1, N=5, B=4, K=3, f_lo=-0.5, f_hi=0.5, r_n=2),
        Cfg("n2", M=2, N=2, B=2, K=2, f_lo=-1.0, f_hi=1.0, r_n=1),
        Cfg("ragged", M=3, N=37, B=8, K=7, f_lo=-2.0, f_hi=3.0, r_n=3),
        C1,
        Cfg("p512", M=2, N=200, B=8, K=9, f_lo=-0.5, f_hi=0.5),
        Cfg("p1024", M=2, N=512, B=8, K=5, f_lo=-256.0, f_hi=256.0),
        Cfg("p2048", M=2, N=1024, B=16, K=3, f_lo=-0.5, f_hi=0.5),
        Cfg("p4096", M=1, N=1500, B=4, K=2, f_lo=-0.5, f_hi=0.5),
        Cfg("p8192", M=1, N=4096, B=16, K=2, f_lo=-0.5, f_hi=0.5),
        Cfg("p8192-m2", M=2, N=3001, B=16, K=3, f_lo=-0.5, f_hi=0.5),     # cross maps at P = 8192, ragged N
        Cfg("batch", M=2, N=48, B=4, K=5, f_lo=-0.5, f_hi=0.5, R=3),
        Cfg("roi", M=2, N=40, B=4, K=5, f_lo=-1.0, f_hi=1.0, tau_lo=-10, tau_hi=25),
    ]


def random_inputs(c, seed):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=seed)
    s = np.exp(2j * np.pi * z.astype(np.float64)).astype(np.complex64)
    w = inputs.random_complex((c.R, c.M, c.N), seed + 100)
    # energy N per row (the feasible set of Eq. 31)
    w = (w * np.sqrt(c.N / np.sum(np.abs(w.astype(np.complex128)) ** 2, axis=-1, keepdims=True))).astype(np.complex64)
    return s, w


def argmax_unique(A_ref, c, auto: bool):
    """Is the oracle's max unique by a relative margin > 1e-5?"""
    v = np.abs(A_ref) / c.N
    M, N = c.M, c.N
    mask = np.zeros_like(v, dtype=bool)
    for m in range(M):
        for l in range(M):
            if (m == l) != auto:
                continue
            mask[:, m, l] = True
    tau = np.arange(-(N - 1), N)
    tlo = c.tlo
    thi = c.thi
    roi = (tau >= tlo) & (tau <= thi)
    mask &= roi[None, None, None, None, :]
    if auto and c.exclude_auto_zero_delay:
        mask[..., N - 1] = False
    vals = np.sort(v[mask])[::-1]
    return len(vals) < 2 or vals[0] - vals[1] > 1e-5 * vals[0]


@pytest.mark.parametrize("c", cases_fwd(), ids=lambda c: c.name)
@pytest.mark.parametrize("mode", [sqngd.LOSS_MAX, sqngd.LOSS_LSE, sqngd.LOSS_PNORM])
def test_forward_map_and_metrics(c, mode):
    c = c.with_(loss_mode=mode, beta_or_p={0: 0.0, 1: 200.0, 2: 16.0}[mode])
    if c.N >= 1500 and mode != sqngd.LOSS_LSE and c.name != "p8192-m2":
        pytest.skip("large-N map checked once")
    s, w = random_inputs(c, 7)
    ctx = sqngd.Context(c)
    met_buf, p, amap = ctx.af_forward(T(s), T(w), want_map=True)
    torch.cuda.synchronize()
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
        assert abs(g["loss_wpsl"] - o["loss_wpsl"]) <= 1e-5 * abs(o["loss_wpsl"])
        assert g["n_cells"] == o["n_cells"]
        if argmax_unique(A[r:r + 1], c, True):
            assert g["argmax_auto"] == o["argmax_auto"]
        if c.M > 1 and argmax_unique(A[r:r + 1], c, False):
            assert g["argmax_cross"] == o["argmax_cross"]
        np.testing.assert_allclose(p.cpu().numpy()[r], ref_p[r], rtol=1e-6, atol=1e-7)


def grad_cases():
    return [
        Cfg("g-tiny", M=2, N=5, B=4, K=3, f_lo=-0.7, f_hi=0.9, r_n=2, eps_w=0.4),
        Cfg("g-ragged", M=3, N=29, B=8, K=5, f_lo=-1.5, f_hi=2.0, r_n=3),
        Cfg("g-c1", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5),
        Cfg("g-p512", M=2, N=256, B=8, K=6, f_lo=-0.5, f_hi=0.5, R=2),
        Cfg("g-p2048", M=2, N=1024, B=16, K=3, f_lo=-0.5, f_hi=0.5),
    ]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("c", grad_cases(), ids=lambda c: c.name)
@pytest.mark.parametrize("mode", [sqngd.LOSS_MAX, sqngd.LOSS_LSE, sqngd.LOSS_PNORM])
def test_gradients_explicit_waveform(c, mode):
    c = c.with_(loss_mode=mode, beta_or_p={0: 0.0, 1: 60.0, 2: 8.0}[mode])
    s, w = random_inputs(c, 11)
    ref_met, gw_ref, gs_ref = O.loss_grad(c, s, w)
    ctx = sqngd.Context(c)
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


@pytest.mark.parametrize("B,r_n,c_", [(4, 3, 300.0), (8, 100, 300.0), (16, 100, 300.0), (4, 2, 30.0)])
def test_quantizer(B, r_n, c_):
    c = Cfg("q", M=3, N=700, B=B, K=1, f_lo=0.0, f_hi=0.0, r_n=r_n, c=c_, R=2)
    z = inputs.phase_params(c.R, c.M, c.N, config_index=3)
    z[0, 0, :5] = [-0.1, 0.0, 1.0, 1.5, 0.5]          # edges / out of range
    rho = inputs.random_sorted_thresholds(c.R, B, r_n, seed=5)
    q = O.quantize(c, z, rho)
    ctx = sqngd.Context(c)
    out = ctx.quantize(T(z), T(rho))
    ctx.sync()
    b = out["b_hard"].cpu().numpy().astype(np.int32)
    assert np.array_equal(b, q["b_hard"]), f"{(b != q['b_hard']).sum()} hard indices differ"
    np.testing.assert_allclose(out["s_hard"].cpu().numpy(), q["s_hard"], atol=2e-7)
    ph = np.angle(out["s_soft"].cpu().numpy().astype(np.complex128) * np.conj(q["s_soft"]))
    record("s_soft phase rad", np.abs(ph).max(), 1e-6)
    assert np.abs(ph).max() < 1e-6, np.abs(ph).max()
    dq = out["dq"].cpu().numpy()
    np.testing.assert_allclose(dq, q["dq"], rtol=2e-5, atol=1e-6 * q["dq"].max())


@pytest.mark.parametrize("mode", [sqngd.LOSS_LSE, sqngd.LOSS_MAX])
def test_transmit_chain_z_rho(mode):
    c = Cfg("chain", M=2, N=48, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=4, c=60.0, loss_mode=mode,
            beta_or_p=60.0 if mode else 0.0, R=2)
    z = inputs.phase_params(c.R, c.M, c.N, config_index=9)
    rho = inputs.random_sorted_thresholds(c.R, c.B, c.r_n, seed=4)
    _, w = random_inputs(c, 21)
    q = O.quantize(c, z, rho)
    _, _, gs = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs)
    ctx = sqngd.Context(c)
    met, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
    ctx.sync()
    check_grad(gz.cpu().numpy(), gz_ref, "grad_z")
    check_grad(gr.cpu().numpy(), gr_ref, "grad_rho")
    # Step A flavour through (z, rho): s_hard then grad_w
    _, gw_ref, _ = O.loss_grad(c, q["s_hard"], w, want_s=False)
    met, gw = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_FILTERS)
    ctx.sync()
    check_grad(gw.cpu().numpy(), gw_ref, "grad_w")


def test_step_teacher_forced_and_invariants():
    """One A+B block: the GPU Adam/projection applied to the GPU gradients equals the
    oracle's Adam/projection applied to the same gradients (teacher forcing, O6)."""
    c = Cfg("step", M=2, N=32, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=4, c=300.0, n_h=1, n_x=1, lr_z=1e-3)
    z = inputs.phase_params(1, c.M, c.N, config_index=12)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    q = O.quantize(c, z, rho)
    w = q["s_hard"].astype(np.complex64)
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z), T(rho), T(w))
    # GPU gradients at the start state, to teacher-force the oracle's Adam
    _, gw = ctx.af_loss_grad(st["z"], st["rho"], st["w"], sqngd.WRT_FILTERS)
    gw = gw.cpu().numpy().astype(np.complex128)
    hist = torch.zeros((1, 2), dtype=torch.float64, device=DEV)     # block A alone fills column 0
    hist_b = torch.zeros((1, 2), dtype=torch.float64, device=DEV)   # block B alone fills column 0
    hard = torch.empty(sqngd.METRICS_BYTES, dtype=torch.uint8, device=DEV)
    st_a = {k: (v.clone() if torch.is_tensor(v) else v) for k, v in st.items()}
    ctx.step(st_a, sqngd.BLOCK_A, hist=hist)
    ctx.sync()
    ost = O.new_state(z, rho, w)
    O.step(c, ost, block=1, grads_from=lambda kind, i, s_: gw)
    np.testing.assert_allclose(st_a["w"].cpu().numpy(), ost["w"], rtol=0, atol=2e-6)
    np.testing.assert_array_equal(st_a["z"].cpu().numpy(), z)          # block isolation
    np.testing.assert_allclose(np.sum(np.abs(st_a["w"].cpu().numpy().astype(np.complex128)) ** 2, -1), c.N,
                               rtol=1e-6)
    # Step B from the post-A state
    _, gz, gr = ctx.af_loss_grad(st_a["z"], st_a["rho"], st_a["w"], sqngd.WRT_TRANSMIT)
    gz, gr = gz.cpu().numpy().astype(np.float64), gr.cpu().numpy().astype(np.float64)
    w_a = st_a["w"].clone()
    z_a, rho_a = st_a["z"].cpu().numpy(), st_a["rho"].cpu().numpy()
    ctx.step(st_a, sqngd.BLOCK_B, hist=hist_b, hard_met=hard)
    ctx.sync()
    ost = O.new_state(st_a["z"].cpu().numpy() * 0 + z, rho, w_a.cpu().numpy())
    O.step(c, ost, block=2, grads_from=lambda kind, i, s_: (gz, gr))
    np.testing.assert_allclose(st_a["z"].cpu().numpy(), ost["z"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(st_a["rho"].cpu().numpy(), ost["rho"], rtol=0, atol=1e-6)
    assert torch.equal(st_a["w"], w_a)                                  # block isolation
    h = np.array([hist.cpu().numpy()[0, 0], hist_b.cpu().numpy()[0, 0]])
    assert np.isfinite(h).all() and (h > 0).all()
    # hard_out: the metrics of the iterate the step started from (explicit forward: no Step A)
    hm = sqngd.metrics_from_bytes(hard.cpu().numpy())[0]
    q2 = O.quantize(c, z_a, rho_a)
    om, _, _ = O.af(c, q2["s_hard"], w_a.cpu().numpy())
    assert abs(hm["wpsl"] - om[0]["wpsl"]) <= 1e-4 * om[0]["wpsl"]
    assert np.isfinite(hm["snrl_db_max"])


def test_determinism():
    c = C1.with_(loss_mode=sqngd.LOSS_LSE, beta_or_p=200.0)
    s, w = random_inputs(c, 3)
    ctx = sqngd.Context(c)
    outs = []
    for _ in range(3):
        met, g = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_TRANSMIT)
        outs.append((met.clone(), g.clone()))
    ctx.sync()
    for m_, g_ in outs[1:]:
        assert torch.equal(m_, outs[0][0]) and torch.equal(g_, outs[0][1])


def test_step_graph_replay_matches_eager():
    """sqngd_step on a side stream is captured into a CUDA graph and replayed; the result must be
    bit-identical to the eager (legacy-stream) execution of the same steps."""
    c = Cfg("graph", M=2, N=48, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=4, n_h=2, n_x=2, lr_z=1e-3)
    z = inputs.phase_params(1, c.M, c.N, config_index=14)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
    ctx = sqngd.Context(c)
    outs = []
    for use_side in (False, True):
        st = ctx.new_state(T(z), T(rho), T(w))
        hist = torch.zeros((1, 4), dtype=torch.float64, device=DEV)
        hard = torch.empty(sqngd.METRICS_BYTES, dtype=torch.uint8, device=DEV)
        stream = torch.cuda.Stream() if use_side else torch.cuda.default_stream()
        with torch.cuda.stream(stream):
            for _ in range(3):  # first call captures, later calls replay
                ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
        torch.cuda.synchronize()
        ctx.sync()
        outs.append((st, hist.clone(), hard.clone()))
    (a, ha, ma), (b, hb, mb) = outs
    for k in ("z", "rho", "w", "m_w", "v_w", "m_z", "v_z", "m_rho", "v_rho"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(ha, hb) and torch.equal(ma, mb)
    assert a["t_a"] == b["t_a"] == 6 and a["t_b"] == b["t_b"] == 6


@pytest.mark.parametrize("engine", [sqngd.ENGINE_FFT, sqngd.ENGINE_CHEBYSHEV])
def test_step_deterministic_with_restarts(engine):
    """R = 2 restarts, R M = 4 filter rows (not a multiple of the row kernel's groups per CTA): the
    same Step-A sequence twice is bit-identical (a padding group once raced on the last row's Adam
    moments)."""
    c = Cfg("detR", M=2, N=32, B=4, K=9, f_lo=-0.5, f_hi=0.5, r_n=4, R=2, n_h=3, n_x=2, lr_w=0.3, lr_z=3e-2,
            doppler_engine=engine)
    z = inputs.phase_params(c.R, c.M, c.N, config_index=31)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
    ctx = sqngd.Context(c)
    outs = []
    for _ in range(2):
        st = ctx.new_state(T(z), T(rho), T(w))
        for _ in range(6):
            ctx.step(st, sqngd.BLOCK_AB)
        outs.append(st)
    ctx.sync()
    for k in ("z", "rho", "w", "m_w", "v_w", "m_z", "v_z", "m_rho", "v_rho"):
        assert torch.equal(outs[0][k], outs[1][k]), k


@pytest.mark.parametrize("mode", [sqngd.LOSS_MAX, sqngd.LOSS_LSE])
def test_correlation_mode_K1(mode):
    """Correlation mode (K = 1, f = 0: the periodic-free aperiodic correlation workload of the
    paper's Table I): map, metrics and both gradients against the oracle."""
    c = Cfg("corr", M=4, N=256, B=8, K=1, f_lo=0.0, f_hi=0.0, r_n=8, loss_mode=mode,
            beta_or_p=200.0 if mode == sqngd.LOSS_LSE else 0.0)
    s, w = random_inputs(c, 41)
    ctx = sqngd.Context(c)
    assert ctx.engine_info()["engine"] == "fft"
    met, _, amap = ctx.af_forward(T(s), T(w), want_map=True)
    m = ctx.metrics(met)[0]
    ref, _, A = O.af(c, s, w, want_A=True)
    check_map(amap.cpu().numpy(), A, c.N)
    assert abs(m["loss"] - ref[0]["loss"]) <= 1e-5 * abs(ref[0]["loss"])
    _, gw = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_FILTERS)
    _, gs = ctx.loss_grad_s(T(s), T(w), sqngd.WRT_TRANSMIT)
    ctx.sync()
    _, gw_ref, gs_ref = O.loss_grad(c, s, w)
    check_grad(gw.cpu().numpy(), gw_ref, "grad_w")
    check_grad(gs.cpu().numpy(), gs_ref, "grad_s")


def test_threshold_projection_with_clusters():
    """Thresholds in clusters of 64 spaced 1e-6 apart (the state long runs reach) with a large rate:
    Adam reorders the clusters, so the projection (Q22: sort, clamp, min-gap sweep) does real work.
    The GPU step (1024-thread projection kernel with the register/shuffle bitonic sort) matches the
    oracle's Adam + projection on the same gradient.  Tolerance 2e-5:
    the fp32 min-gap sweep accumulates 1e-6 steps along a 64-long cluster."""
    c = Cfg("clus", M=2, N=64, B=16, K=9, f_lo=-0.5, f_hi=0.5, r_n=100, n_h=1, n_x=1, lr_z=1e-2,
            doppler_engine=sqngd.ENGINE_FFT)
    z = inputs.phase_params(1, c.M, c.N, config_index=17)
    base = inputs.init_thresholds(1, c.B, c.r_n).astype(np.float64)[0]
    rho = base.copy()
    for g0 in range(0, c.BR, 64):  # squeeze each group of 64 around its mean
        grp = slice(g0, min(g0 + 64, c.BR))
        n = grp.stop - grp.start
        rho[grp] = base[grp].mean() + (np.arange(n) - n / 2) * 1e-6
    rho = rho.astype(np.float32)[None]
    assert (np.diff(rho[0]) > 0).all()
    w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z), T(rho), T(w))
    _, gz, gr = ctx.af_loss_grad(st["z"], st["rho"], st["w"], sqngd.WRT_TRANSMIT)
    ctx.sync()
    gz, gr = gz.cpu().numpy().astype(np.float64), gr.cpu().numpy().astype(np.float64)
    ctx.step(st, sqngd.BLOCK_B)
    ctx.sync()
    ost = O.new_state(z, rho, w)
    O.step(c, ost, block=2, grads_from=lambda kind, i, s_: (gz, gr))
    r_gpu = st["rho"].cpu().numpy()
    assert (np.diff(r_gpu[0]) >= 0).all()
    np.testing.assert_allclose(r_gpu, ost["rho"], rtol=0, atol=2e-5)
    # the oracle's update did reorder thresholds (the sort was exercised)
    raw = rho.astype(np.float64) - 1e-2 * np.sign(gr)
    assert (np.diff(raw[0]) < 0).any()


def test_grad_rho_clustered_z_multichunk():
    """k_grad_rho (one pass, window compaction per 4096-element chunk): z clustered in a narrow band so
    every threshold block's window union holds whole chunks (MN = 2 x 2600 -> two chunks, the second
    ragged), thresholds clustered around the band; grad_z / grad_rho against the oracle chain (Eq. 25)."""
    c = Cfg("rhoclu", M=2, N=2600, B=8, K=3, f_lo=-0.5, f_hi=0.5, r_n=24, c=300.0,
            loss_mode=sqngd.LOSS_LSE, beta_or_p=60.0)
    rng = np.random.default_rng(77)
    z = (0.5 + 0.01 * (rng.random((1, c.M, c.N)) - 0.5)).astype(np.float32)
    rho = np.sort(0.5 + 0.02 * (rng.random((1, c.B * c.r_n)) - 0.5)).astype(np.float32)
    _, w = random_inputs(c, 5)
    q = O.quantize(c, z, rho)
    _, _, gs = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs)
    ctx = sqngd.Context(c)
    met, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
    ctx.sync()
    check_grad(gz.cpu().numpy(), gz_ref, "grad_z (clustered z)")
    check_grad(gr.cpu().numpy(), gr_ref, "grad_rho (clustered z, 2 chunks)")
