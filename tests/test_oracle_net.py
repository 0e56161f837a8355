"""Pins of the generator oracle z = f_theta(y0) (oracle/net_oracle.py; Eq. 20 P:L223-227,
P:L583).  Each pin is independent of the oracle's own backward code:
central finite differences of its forward, structural identities of the architecture (the
residual identity path, the closed-form parameter count), and the end-to-end chain through the
AF loss (finite differences of the full pipeline, SPEC generator-net invariant)."""
import os
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import net_oracle as NO
from oracle import oracle as O
from paper_2604_25728_b200 import inputs


def rnd_theta(Din, W, D, seed, scale=0.6):
    g = np.random.default_rng(seed)
    return g.standard_normal(NO.num_params(Din, W, D)) * scale


def test_parameter_count_closed_form():
    # SPEC generator-net: D (2 W^2 + 2 W) + input/output affine counts
    for Din, W, D in [(12, 8, 2), (8192, 128, 5), (65536, 128, 5), (3, 1, 0)]:
        assert NO.num_params(Din, W, D) == D * (2 * W * W + 2 * W) + (W * Din + W) + (Din * W + Din)
    # the paper's C3 generator: 5 blocks, width 128, M N = 8192 inputs
    assert NO.num_params(8192, 128, 5) == 2_270_592
    th = inputs.net_params(1, 40, 32, 3)
    assert th.shape == (1, NO.num_params(40, 32, 3))
    th = inputs.net_params(1, 111, 16, 1)  # Din % 4 = 3: one pad float to the float4 stride
    assert th.shape == (1, NO.num_params(111, 16, 1) + 1) and th[0, -1] == 0


def test_gradients_match_central_differences():
    """Every parameter and input entry of a width-8 depth-2 instance (SPEC's FD example)."""
    Din, W, D = 6, 8, 2
    th = rnd_theta(Din, W, D, 1)
    y0 = np.random.default_rng(2).random(Din)
    gz = np.random.default_rng(3).standard_normal(Din)
    z, tape = NO.forward(th, y0, Din, W, D)
    g, gy = NO.backward(th, tape, gz, Din, W, D)

    def L(t, y):
        return float(NO.forward(t, y, Din, W, D)[0] @ gz)

    h = 1e-6
    fd = np.empty_like(th)
    for i in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        fd[i] = (L(tp, y0) - L(tm, y0)) / (2 * h)
    scale = np.abs(fd).max()
    assert np.abs(fd - g).max() < 1e-7 * scale, np.abs(fd - g).max() / scale
    fdy = np.array([(L(th, y0 + h * e) - L(th, y0 - h * e)) / (2 * h) for e in np.eye(Din)])
    assert np.abs(fdy - gy).max() < 1e-7 * np.abs(fdy).max()
    # every parameter group actually receives gradient (no dropped term)
    gp = NO.unpack(g, Din, W, D)
    for name in ("W_in", "b_in", "W_out", "b_out"):
        assert np.abs(gp[name]).max() > 1e-6, name
    for b in gp["blocks"]:
        for name in ("W1", "b1", "W2", "b2"):
            assert np.abs(b[name]).max() > 1e-6, name


def test_zero_inner_weights_is_the_identity_path():
    """SPEC generator-net: zero inner weights -> residual blocks act as identity, so the
    network equals the depth-0 network with the same input/output affine maps."""
    Din, W, D = 10, 8, 3
    th = rnd_theta(Din, W, D, 4)
    p = NO.unpack(th, Din, W, D)
    for b in p["blocks"]:
        for k in ("W1", "b1", "W2", "b2"):
            b[k][...] = 0.0
    th0 = np.concatenate([p["W_in"].ravel(), p["b_in"], p["W_out"].ravel(), p["b_out"]])
    y0 = np.random.default_rng(5).random(Din)
    z, _ = NO.forward(th, y0, Din, W, D)
    z0, _ = NO.forward(th0, y0, Din, W, 0)
    np.testing.assert_array_equal(z, z0)
    # and with W_in = 0, b_in = 0 (h_0 = 0) the output is sigmoid(b_out): W_out sees a zero vector
    p["W_in"][...] = 0.0
    p["b_in"][...] = 0.0
    z1, _ = NO.forward(th, y0, Din, W, D)
    np.testing.assert_allclose(z1, 0.5 * (1.0 + np.tanh(p["b_out"] / 2.0)), rtol=1e-15)


def test_output_range_and_linearity_of_adjoint():
    Din, W, D = 9, 8, 2
    th = rnd_theta(Din, W, D, 6, scale=0.8)
    y0 = np.random.default_rng(7).random(Din)
    z, tape = NO.forward(th, y0, Din, W, D)
    assert ((z > 0) & (z < 1)).all()
    g1, _ = NO.backward(th, tape, np.ones(Din), Din, W, D)
    g2, _ = NO.backward(th, tape, np.arange(Din, dtype=float), Din, W, D)
    g3, _ = NO.backward(th, tape, np.ones(Din) + 2 * np.arange(Din), Din, W, D)
    np.testing.assert_allclose(g3, g1 + 2 * g2, rtol=1e-12, atol=1e-14)
    g0, gy0 = NO.backward(th, tape, np.zeros(Din), Din, W, D)
    assert not g0.any() and not gy0.any()


def test_seeded_init_statistics():
    """SPEC generator-net init example: for N M = 1024 the initial output std lies in [0.05, 0.45]
    and every output is inside (0, 1); same seed -> identical parameters."""
    Din, W, D = 1024, 128, 5
    th = inputs.net_params(1, Din, W, D, config_index=3)
    np.testing.assert_array_equal(th, inputs.net_params(1, Din, W, D, config_index=3))
    y0 = inputs.net_input(1, 4, 256, 8, config_index=3)
    assert set(np.unique(y0 * 8).astype(int)) <= set(range(8))
    z, _ = NO.forward(th[0].astype(np.float64), y0[0], Din, W, D)
    assert ((z > 0) & (z < 1)).all() and 0.05 <= z.std() <= 0.45


def test_end_to_end_chain_through_the_af_loss():
    """SPEC generator-net invariant: d loss / d theta through the generator, the soft quantizer
    (Eqs. 21-24) and the AF loss (Eqs. 7-10, 37-42, LSE) matches central differences of the
    full pipeline at N <= 16, M <= 2."""
    c = SimpleNamespace(R=1, M=2, N=6, B=4, r_n=2, c=20.0, K=3, f_lo=-0.5, f_hi=0.5, tau_lo=None, tau_hi=None,
                        exclude_auto_zero_delay=1, loss_mode=1, beta_or_p=15.0, eps_w=0.4, mu_db=0.5)
    Din, W, D = c.M * c.N, 8, 2
    th = rnd_theta(Din, W, D, 8, scale=0.5)
    y0 = inputs.net_input(1, c.M, c.N, c.B, config_index=9)[0].astype(np.float64)
    rho = ((np.arange(8) + 0.5) / 8 + 0.01 * np.sin(np.arange(8))).reshape(1, -1)
    w = np.exp(2j * np.pi * np.random.default_rng(10).random((1, c.M, c.N)))

    def L(t):
        z, _ = NO.forward(t, y0, Din, W, D)
        q = O.quantize(c, z.reshape(1, c.M, c.N), rho)
        return O.af(c, q["s_soft"], w)[0][0]["loss"]

    z, tape = NO.forward(th, y0, Din, W, D)
    q = O.quantize(c, z.reshape(1, c.M, c.N), rho)
    _, _, gs = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz, _ = O.chain(c, z.reshape(1, c.M, c.N), rho, q["s_soft"], gs)
    g, _ = NO.backward(th, tape, gz.reshape(Din), Din, W, D)
    h = 1e-6
    idx = np.random.default_rng(11).choice(th.size, 40, replace=False)
    scale = np.abs(g).max()
    for i in idx:
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        assert abs((L(tp) - L(tm)) / (2 * h) - g[i]) < 1e-3 * scale


def test_oracle_step_generator_mode():
    """Alg. 1 with z = f_theta(y0): Step A leaves theta alone, Step B moves theta
    (not z directly), and the returned z is f_theta(y0) of the returned theta."""
    c = SimpleNamespace(R=1, M=2, N=8, B=4, r_n=2, c=30.0, K=3, f_lo=-0.5, f_hi=0.5, tau_lo=None, tau_hi=None,
                        exclude_auto_zero_delay=1, loss_mode=1, beta_or_p=20.0, eps_w=0.1, mu_db=0.5,
                        lr_w=5e-2, lr_z=1e-4, lr_theta=1e-3, adam_b1=0.9, adam_b2=0.999, adam_eps=1e-8,
                        n_h=2, n_x=3, net_width=8, net_depth=2)
    Din = c.M * c.N
    th = inputs.net_params(1, Din, 8, 2, config_index=4)[:, :NO.num_params(Din, 8, 2)]
    y0 = inputs.net_input(1, c.M, c.N, c.B, config_index=4)
    z0, _ = NO.forward(th[0].astype(np.float64), y0[0], Din, 8, 2)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    w = np.exp(2j * np.pi * np.random.default_rng(12).random((1, c.M, c.N)))
    st = O.new_state(z0.reshape(1, c.M, c.N), rho, w, theta=th, y0=y0)
    O.step(c, st, block=1)
    np.testing.assert_array_equal(st["theta"], th.astype(np.float64))
    hist = O.step(c, st, block=2)
    assert hist.shape == (3, 1) and np.isfinite(hist).all()
    assert np.abs(st["theta"] - th).max() > 1e-4
    zf, _ = NO.forward(st["theta"][0], y0[0], Din, 8, 2)
    np.testing.assert_array_equal(st["z"].reshape(-1), zf)
