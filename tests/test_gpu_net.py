"""Generator z = f_theta(y0) through the C-ABI vs the fp64 oracle
(oracle/net_oracle.py) on identical seeded fp32 inputs.

Tolerances:
  z:          |z_gpu - z_ref| <= 2e-5  (fp32 dot products of Din <= 65536 terms feed a sigmoid
                                        whose slope is <= 1/4; measured worst ~1e-6)
  gradients:  normwise relative error of every parameter group <= 1e-4 (the AF gradients' bar)
  Adam step:  teacher forced with the GPU's own gradient; |theta_gpu - theta_ref| <= 1e-6 + lr
              (one fp32 Adam step moves each entry by at most ~lr)
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import net_oracle as NO  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import C3, C5, Cfg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def T(a, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV, dtype=dtype)


def groups(g, Din, W, D):
    p = NO.unpack(g, Din, W, D)
    out = {"W_in": p["W_in"], "b_in": p["b_in"], "W_out": p["W_out"], "b_out": p["b_out"]}
    for d, b in enumerate(p["blocks"]):
        for k, v in b.items():
            out[f"{k}_{d}"] = v
    return out


def rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300)


CASES = [
    # name, cfg, W, D
    ("small", Cfg("n_small", M=2, N=32, B=4, K=3, f_lo=-0.5, f_hi=0.5, r_n=2), 32, 2),
    ("ragged", Cfg("n_rag", M=3, N=37, B=8, K=3, f_lo=-0.5, f_hi=0.5, r_n=2, R=2), 16, 1),  # Din = 111, R = 2
    ("depth0", Cfg("n_d0", M=2, N=64, B=4, K=3, f_lo=-0.5, f_hi=0.5, r_n=2), 8, 0),
    ("w128_tail", Cfg("n_tail", M=1, N=300, B=4, K=3, f_lo=-0.5, f_hi=0.5, r_n=2), 128, 3),  # Din % 256 != 0
    ("C3", C3, 128, 5),
    ("C5_R2", C5.with_(R=2), 128, 5),
]


@pytest.mark.parametrize("name,c,W,D", CASES, ids=[x[0] for x in CASES])
def test_forward_backward_parity(name, c, W, D):
    c = c.with_(net_width=W, net_depth=D)
    Din = c.M * c.N
    th = inputs.net_params(c.R, Din, W, D, config_index=7, bias_scale=0.1)
    y0 = inputs.net_input(c.R, c.M, c.N, c.B, config_index=7)
    gz = inputs.uniform01_f32(77, c.R * Din).reshape(c.R, Din) - np.float32(0.5)
    ctx = sqngd.Context(c)
    dth, dy0 = T(th), T(y0)
    z = ctx.net_forward(dth, dy0)
    g = ctx.net_backward(dth, dy0, z, T(gz.reshape(c.R, c.M, c.N)))
    ctx.sync()
    z = z.cpu().numpy().reshape(c.R, Din)
    g = g.cpu().numpy()
    zr, tapes = NO.forward_batch(th.astype(np.float64), y0, Din, W, D)
    assert np.abs(z - zr).max() <= 2e-5, np.abs(z - zr).max()
    gr = NO.backward_batch(th.astype(np.float64), tapes, gz, Din, W, D)
    for r in range(c.R):
        G, Gr = groups(g[r], Din, W, D), groups(gr[r], Din, W, D)
        for k in Gr:
            assert rel(G[k], Gr[k]) <= 1e-4, (r, k, rel(G[k], Gr[k]))


def test_backward_deterministic_and_theta_untouched():
    c = CASES[0][1].with_(net_width=32, net_depth=2, R=2)
    Din = c.M * c.N
    th = T(inputs.net_params(c.R, Din, 32, 2, config_index=8))
    y0 = T(inputs.net_input(c.R, c.M, c.N, c.B, config_index=8))
    ctx = sqngd.Context(c)
    outs = []
    for _ in range(3):
        z = ctx.net_forward(th, y0)
        outs.append((z.clone(), ctx.net_backward(th, y0, z, torch.ones_like(z)).clone()))
    ctx.sync()
    for zz, gg in outs[1:]:
        assert torch.equal(zz, outs[0][0]) and torch.equal(gg, outs[0][1])
    assert torch.equal(th, T(inputs.net_params(c.R, Din, 32, 2, config_index=8)))


def test_no_generator_is_invalid():
    ctx = sqngd.Context(CASES[0][1])
    with pytest.raises(sqngd.SqngdError) as e:
        ctx.net_forward(torch.zeros(10, device=DEV), torch.zeros(64, device=DEV))
    assert e.value.status == sqngd.E_INVALID


def _net_state(c, W, D, idx):
    Din = c.M * c.N
    th = inputs.net_params(c.R, Din, W, D, config_index=idx)
    y0 = inputs.net_input(c.R, c.M, c.N, c.B, config_index=idx)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    z0 = np.stack([NO.forward(th[r].astype(np.float64), y0[r], Din, W, D)[0] for r in range(c.R)])
    z0 = z0.reshape(c.R, c.M, c.N).astype(np.float32)
    w = O.quantize(c, z0, rho)["s_hard"].astype(np.complex64)
    return th, y0, rho, z0, w


@pytest.mark.parametrize("engine", [sqngd.ENGINE_FFT, sqngd.ENGINE_CHEBYSHEV])
def test_step_B_teacher_forced(engine):
    """One Step-B inner step in generator mode: the GPU's fused backward + Adam(theta) equals the
    oracle's Adam applied to the GPU's own dL/dtheta (teacher forcing), rho likewise, and the
    returned z is f_theta(y0) of the returned theta."""
    W, D = 32, 2
    c = Cfg("n_step", M=2, N=48, B=4, K=7, f_lo=-0.5, f_hi=0.5, r_n=4, n_h=1, n_x=1, lr_theta=1e-3,
            lr_z=1e-3, net_width=W, net_depth=D, doppler_engine=engine)
    th, y0, rho, z0, w = _net_state(c, W, D, 21)
    Din = c.M * c.N
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z0), T(rho), T(w), theta=T(th), y0=T(y0))
    # the GPU's gradients at the start state
    z = ctx.net_forward(st["theta"], st["y0"])
    _, gz, gr = ctx.af_loss_grad(z, st["rho"], st["w"], sqngd.WRT_TRANSMIT)
    gth = ctx.net_backward(st["theta"], st["y0"], z, gz)
    ctx.sync()
    gth, gr = gth.cpu().numpy().astype(np.float64), gr.cpu().numpy().astype(np.float64)
    hist = torch.zeros((1, 1), dtype=torch.float64, device=DEV)
    ctx.step(st, sqngd.BLOCK_B, hist=hist)
    ctx.sync()
    ost = O.new_state(z.cpu().numpy(), rho, w, theta=th, y0=y0)
    oc = c
    O.step(oc, ost, block=2, grads_from=lambda kind, i, s_: (gth, gr))
    tg = st["theta"].cpu().numpy()
    assert np.abs(tg - ost["theta"]).max() <= 1e-6 + 1e-5, np.abs(tg - ost["theta"]).max()
    np.testing.assert_allclose(st["rho"].cpu().numpy(), ost["rho"], rtol=0, atol=1e-6)
    assert np.abs(tg - th).max() > 5e-4  # theta moved by ~lr
    zr = np.stack([NO.forward(tg[r].astype(np.float64), y0[r], Din, W, D)[0] for r in range(c.R)])
    assert np.abs(st["z"].cpu().numpy().reshape(c.R, Din) - zr).max() <= 2e-5
    h = hist.cpu().numpy()
    assert np.isfinite(h).all() and h[0, 0] > 0


def test_step_graph_replay_matches_eager_generator():
    W, D = 16, 1
    c = Cfg("n_graph", M=2, N=40, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=4, n_h=2, n_x=2, lr_theta=1e-3,
            net_width=W, net_depth=D)
    th, y0, rho, z0, w = _net_state(c, W, D, 22)
    ctx = sqngd.Context(c)
    outs = []
    for use_side in (False, True):
        st = ctx.new_state(T(z0), T(rho), T(w), theta=T(th), y0=T(y0))
        hist = torch.zeros((1, 4), dtype=torch.float64, device=DEV)
        stream = torch.cuda.Stream() if use_side else torch.cuda.default_stream()
        with torch.cuda.stream(stream):
            for _ in range(3):
                ctx.step(st, sqngd.BLOCK_AB, hist=hist)
        torch.cuda.synchronize()
        ctx.sync()
        outs.append((st, hist.clone()))
    (a, ha), (b, hb) = outs
    for k in ("z", "rho", "w", "theta", "m_theta", "v_theta", "m_rho", "v_rho", "m_w", "v_w"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(ha, hb)
    assert not torch.equal(a["theta"], T(th))


def test_C3_generator_step_runs():
    """The paper's generator (5 blocks, width 128) on C3 with the default engine: one
    outer iteration, finite losses, z = f_theta(y0) on return, and the hard PSL reported."""
    W, D = 128, 5
    c = C3.with_(net_width=W, net_depth=D, lr_theta=1e-5)
    th, y0, rho, z0, w = _net_state(c, W, D, 23)
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z0), T(rho), T(w), theta=T(th), y0=T(y0))
    hist = torch.zeros((1, 20), dtype=torch.float64, device=DEV)
    hard = torch.empty(sqngd.METRICS_BYTES, dtype=torch.uint8, device=DEV)
    ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
    ctx.sync()
    h = hist.cpu().numpy()[0]
    assert np.isfinite(h).all() and (h > 0).all()
    Din = c.M * c.N
    zr = NO.forward(st["theta"].cpu().numpy()[0].astype(np.float64), y0[0], Din, W, D)[0]
    assert np.abs(st["z"].cpu().numpy().reshape(Din) - zr).max() <= 2e-5
    m = sqngd.metrics_from_bytes(hard.cpu().numpy())[0]
    assert 0 < m["wpsl"] < 1


def test_hidden_chain_paper_size():
    """The hidden layers on the 8-CTA cluster (DSMEM exchanges) at the paper's 5 x 128, R = 2, against the
    oracle."""
    c = Cfg("n_var", M=4, N=256, B=8, K=3, f_lo=-0.5, f_hi=0.5, r_n=2, R=2, net_width=128, net_depth=5)
    Din = c.M * c.N
    th = inputs.net_params(c.R, Din, 128, 5, config_index=9, bias_scale=0.1)
    y0 = inputs.net_input(c.R, c.M, c.N, c.B, config_index=9)
    gz = inputs.uniform01_f32(99, c.R * Din).reshape(c.R, Din) - np.float32(0.5)
    ctx = sqngd.Context(c)
    z = ctx.net_forward(T(th), T(y0))
    g = ctx.net_backward(T(th), T(y0), z, T(gz.reshape(c.R, c.M, c.N)))
    ctx.sync()
    zr, tapes = NO.forward_batch(th.astype(np.float64), y0, Din, 128, 5)
    assert np.abs(z.cpu().numpy().reshape(c.R, Din) - zr).max() <= 2e-5
    gr = NO.backward_batch(th.astype(np.float64), tapes, gz, Din, 128, 5)
    assert rel(g.cpu().numpy(), gr) <= 1e-4
