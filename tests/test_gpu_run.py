"""Alg. 1 driver sqngd_run through the C-ABI.

The reference is the oracle's stopping_check (O6: the stopping rule and best-snapshot rule of
P:L485 / SPEC S:L542-545, pinned by SPEC's examples in tests/test_oracle_quant_grad.py) applied to
the hard-WPSL history the driver reports, plus a replay: the driver's best snapshot must be
bit-identical to the state after best_iter plain sqngd_step(A+B) calls from the same start
(the steps are deterministic)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def setup(c, idx):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=idx)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
    return [torch.as_tensor(a, device=DEV) for a in (z, rho, w)]


@pytest.mark.parametrize("patience,check_every,need_dec", [(2, 1, False), (3, 4, False), (0, 1, False), (2, 1, True),
                                                        (3, 2, True)])
def test_run_rule_and_snapshot(patience, check_every, need_dec):
    c = Cfg("run", M=2, N=32, B=4, K=9, f_lo=-0.5, f_hi=0.5, r_n=4, R=2, n_h=2, n_x=2, lr_w=0.3, lr_z=3e-2)
    T = 16
    ctx = sqngd.Context(c)
    z, rho, w = setup(c, 31)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        st = ctx.new_state(z, rho, w)
        best, bw, bi, hist, res = ctx.run(st, T=T, patience=patience, check_every=check_every,
                                          require_loss_decrease=need_dec)
    torch.cuda.synchronize()
    h = hist.cpu().numpy()
    lh = res["loss_hist"].cpu().numpy()
    stop, bi_ref, bw_ref = O.stopping_check(np.nan_to_num(h, nan=math.inf)[: res["iterations"]], patience,
                                lh[: res["iterations"]] if need_dec else None)
    if patience > 0 and stop is not None:
        assert res["stopped"] and res["iterations"] == stop
        # iterate t is scored by step t + 1 (hard_out = the entry iterate), so the rule is seen one step later
        assert res["iterations"] <= res["steps_run"] <= res["iterations"] + check_every
        assert np.isnan(h[res["iterations"]:]).all()  # no history past the stop
    else:
        assert not res["stopped"] and res["iterations"] == T
    np.testing.assert_array_equal(bi.cpu().numpy(), bi_ref)
    np.testing.assert_array_equal(bw.cpu().numpy(), bw_ref)
    assert np.isfinite(h[: res["iterations"]]).all() and (h[: res["iterations"]] > 0).all()
    # replay: the snapshot of restart r is the state after bi[r] outer iterations (the same launch
    # sequence as the driver's: every step also evaluates the hard metrics)
    # and every reported history entry is the hard metrics of that iterate: an independent forward
    # (sqngd_af_forward on the iterate's hard waveform) and the next step's hard_out (entry iterate)
    hard = torch.empty(c.R * sqngd.METRICS_BYTES, dtype=torch.uint8, device=DEV)
    n_it = res["iterations"]
    with torch.cuda.stream(side):
        st2 = ctx.new_state(z, rho, w)
        snaps, fwd, entry = {}, [], []
        for t in range(1, max(int(bi_ref.max()), n_it) + 1):
            ctx.step(st2, sqngd.BLOCK_AB, hard_met=hard)
            if t >= 2:
                entry.append([m["wpsl"] for m in sqngd.metrics_from_bytes(hard.cpu().numpy())])
            s_h = ctx.quantize(st2["z"], st2["rho"], soft=False, want_b=False, want_dq=False)["s_hard"]
            met, _, _ = ctx.af_forward(s_h, st2["w"])
            fwd.append([m["wpsl"] for m in ctx.metrics(met)])
            for r in range(c.R):
                if bi_ref[r] == t:
                    snaps[r] = {k: st2[k][r].clone() for k in ("z", "rho", "w")}
    torch.cuda.synchronize()
    for r in range(c.R):
        for k in ("z", "rho", "w"):
            assert torch.equal(best[k][r], snaps[r][k]), (r, k)
    fwd = np.array(fwd)[:n_it]
    np.testing.assert_allclose(h[:n_it], fwd, rtol=1e-6)
    if len(entry):
        np.testing.assert_allclose(np.array(entry)[: n_it - 1], fwd[: len(entry)][: n_it - 1], rtol=1e-6)


def test_run_generator_mode_snapshot_has_theta():
    c = Cfg("run_net", M=2, N=32, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=4, n_h=1, n_x=2, lr_theta=1e-3,
            net_width=16, net_depth=1)
    ctx = sqngd.Context(c)
    th = torch.as_tensor(inputs.net_params(1, c.M * c.N, 16, 1, config_index=5), device=DEV)
    y0 = torch.as_tensor(inputs.net_input(1, c.M, c.N, c.B, config_index=5), device=DEV)
    z = ctx.net_forward(th, y0)
    rho = torch.as_tensor(inputs.init_thresholds(1, c.B, c.r_n), device=DEV)
    w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
    st = ctx.new_state(z, rho, w, theta=th, y0=y0)
    best, bw, bi, hist, res = ctx.run(st, T=6, patience=0)
    ctx.sync()
    assert res["iterations"] == 6 and not res["stopped"]
    b = int(bi.cpu().numpy()[0])
    assert 1 <= b <= 6
    assert bw.cpu().numpy()[0] == np.min(hist.cpu().numpy()[:, 0])
    # the snapshot's z is the generator output of the snapshot's theta
    z2 = ctx.net_forward(best["theta"], y0)
    ctx.sync()
    assert torch.equal(z2, best["z"])


def test_alg1_improves_hard_psl():
    """NEXT-3 trend check: from the seeded matched start, 60 outer iterations of
    Alg. 1 at C1 lower the hard-waveform PSL by more than 3 dB (measured: -11.6 -> -17.4 dB)."""
    from paper_2604_25728_b200.configs import C1

    c = C1.with_(loss_mode=sqngd.LOSS_LSE, beta_or_p=200.0)
    ctx = sqngd.Context(c)
    z = torch.as_tensor(inputs.phase_params(1, c.M, c.N, c.index), device=DEV)
    rho = torch.as_tensor(inputs.init_thresholds(1, c.B, c.r_n), device=DEV)
    w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
    met, _, _ = ctx.af_forward(w, w)
    start = ctx.metrics(met)[0]["wpsl"]
    st = ctx.new_state(z, rho, w)
    best, bw, bi, hist, res = ctx.run(st, T=60, patience=0)
    ctx.sync()
    assert 20 * math.log10(float(bw.cpu()[0])) < 20 * math.log10(start) - 3.0
    # the snapshot is consistent: its hard waveform evaluates to the recorded best WPSL
    q = ctx.quantize(best["z"], best["rho"], soft=False, want_b=False, want_dq=False)
    met, _, _ = ctx.af_forward(q["s_hard"], best["w"])
    assert ctx.metrics(met)[0]["wpsl"] == float(bw.cpu()[0])


def _best_pslr(c, T=60, seed=7):
    """Mean over the restarts of the Alg.-1 best snapshot's hard PSLR (Eq. 48), matched start."""
    ctx = sqngd.Context(c)
    z = torch.as_tensor(inputs.phase_params(c.R, c.M, c.N, config_index=seed), device=DEV)
    rho = torch.as_tensor(inputs.init_thresholds(c.R, c.B, c.r_n), device=DEV)
    w = ctx.quantize(z, rho, soft=False, want_b=False, want_dq=False)["s_hard"]
    st = ctx.new_state(z, rho, w)
    best, bw, bi, hist, res = ctx.run(st, T=T, patience=0, want_hist=False)
    ctx.sync()
    return float(np.mean(20 * np.log10(bw.cpu().numpy())))


def test_trend_table2_snrl_relaxation():
    """NEXT-3 reduced-T trend: the direction of PAPER.md Table II: a larger SNRL
    allowance mu (Eq. 39, p_tar = 10^{-mu/20}) lets the filters trade mainlobe for sidelobes, so the
    best hard PSL falls as mu grows (paper, M=2 N=512 B=4: -24.10 / -29.63 / -32.32 / -33.11 dB at
    mu = 0 / 0.5 / 1 / 1.5).  Here C1 shape, 4 restarts, T = 60 (profiles/r02_trend_tables_II_III.json:
    -16.09 / -17.38 / -17.85 / -18.10 dB)."""
    from paper_2604_25728_b200.configs import C1

    base = C1.with_(R=4, loss_mode=sqngd.LOSS_LSE, beta_or_p=200.0)
    p = {mu: _best_pslr(base.with_(mu_db=mu)) for mu in (0.0, 0.5, 1.0, 1.5)}
    assert p[0.0] > p[0.5] + 0.5 > p[1.5] + 0.5, p
    assert p[1.0] < p[0.5] and p[1.5] <= p[1.0] + 0.05, p


def test_trend_table3_doppler_range():
    """The direction of PAPER.md Table III: a wider Doppler range is harder, so the best hard
    PSL rises with it (paper: -48.87 / -43.09 / -36.10 dB for f in [-0.1, 0.1] / [-0.5, 0.5] / [-3, 3]).
    Here C1 shape, 4 restarts, T = 60 (-19.07 / -17.38 / -14.91 dB)."""
    from paper_2604_25728_b200.configs import C1

    base = C1.with_(R=4, loss_mode=sqngd.LOSS_LSE, beta_or_p=200.0)
    p = {f: _best_pslr(base.with_(f_lo=-f, f_hi=f)) for f in (0.1, 0.5, 3.0)}
    assert p[0.1] + 0.5 < p[0.5] < p[3.0] - 0.5, p
