"""Device-side error statuses through the C-ABI (include/sqngd.h): latched conditions are
returned by sqngd_sync, and sqngd_step keeps the last finite iterate."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
ENGINES = [sqngd.ENGINE_FFT, sqngd.ENGINE_CHEBYSHEV]


def T(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


def cfg(engine, **kw):
    return Cfg("st", M=2, N=48, B=4, K=31, f_lo=-0.5, f_hi=0.5, r_n=4, loss_mode=sqngd.LOSS_LSE, beta_or_p=60.0,
               doppler_engine=engine, n_h=1, n_x=1, **kw)


def sw(c, seed=3):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=seed)
    s = np.exp(2j * np.pi * z.astype(np.float64)).astype(np.complex64)
    return z, s, s.copy()


def expect(ctx, status):
    with pytest.raises(sqngd.SqngdError) as ei:
        ctx.sync()
    assert ei.value.status == status, (ei.value.status, str(ei.value))
    ctx.sync()  # the latch is cleared by the read


@pytest.mark.parametrize("engine", ENGINES)
def test_zero_filter_row_is_degenerate(engine):
    """|w_m^H s_m| = 0 (Eq. 38 undefined for the SNRL term): E_DEGENERATE."""
    c = cfg(engine)
    _, s, w = sw(c)
    w[0, 1] = 0
    ctx = sqngd.Context(c)
    ctx.af_forward(T(s), T(w))
    expect(ctx, sqngd.E_DEGENERATE)


@pytest.mark.parametrize("engine", ENGINES)
def test_nan_input_is_nonfinite(engine):
    c = cfg(engine)
    _, s, w = sw(c)
    w[0, 0, 5] = np.nan
    ctx = sqngd.Context(c)
    ctx.loss_grad_s(T(s), T(w), sqngd.WRT_TRANSMIT)
    expect(ctx, sqngd.E_NONFINITE)


def test_unsorted_thresholds_are_invalid():
    c = cfg(sqngd.ENGINE_FFT)
    z, _, _ = sw(c)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    rho[0, [3, 4]] = rho[0, [4, 3]]
    ctx = sqngd.Context(c)
    ctx.quantize(T(z), T(rho))
    expect(ctx, sqngd.E_INVALID)


@pytest.mark.parametrize("engine", ENGINES)
def test_step_keeps_last_finite_iterate(engine):
    """A non-finite gradient latches E_NONFINITE and sqngd_step applies no update."""
    c = cfg(engine)
    z, _, w = sw(c)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    w[0, 0, 7] = np.inf
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z), T(rho), T(w))
    z0, rho0, w0 = st["z"].clone(), st["rho"].clone(), st["w"].clone()
    ctx.step(st, sqngd.BLOCK_AB)
    expect(ctx, sqngd.E_NONFINITE)
    assert torch.equal(st["z"], z0) and torch.equal(st["rho"], rho0)
    assert torch.equal(torch.view_as_real(st["w"]).nan_to_num(), torch.view_as_real(w0).nan_to_num())


@pytest.mark.parametrize("engine", ENGINES)
def test_generator_step_keeps_last_finite_iterate(engine):
    """Generator mode (NEXT-2): a non-finite gradient latches E_NONFINITE and neither theta, its
    Adam moments nor rho move (the generator backward runs on a forked branch in the graph)."""
    c = cfg(engine, net_width=16, net_depth=1, lr_theta=1e-3)
    z, _, w = sw(c)
    rho = inputs.init_thresholds(1, c.B, c.r_n)
    w[0, 0, 7] = np.inf
    th = T(inputs.net_params(1, c.M * c.N, 16, 1, config_index=6))
    y0 = T(inputs.net_input(1, c.M, c.N, c.B, config_index=6))
    ctx = sqngd.Context(c)
    st = ctx.new_state(T(z), T(rho), T(w), theta=th, y0=y0)
    th0, rho0 = st["theta"].clone(), st["rho"].clone()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):  # graph-captured step (forked generator branch)
        ctx.step(st, sqngd.BLOCK_B)
    side.synchronize()
    expect(ctx, sqngd.E_NONFINITE)
    assert torch.equal(st["theta"], th0) and torch.equal(st["rho"], rho0)
    assert not st["m_theta"].any() and not st["v_theta"].any()


def test_binding_rejects_wrong_dtypes():
    """The C-ABI takes raw pointers: the binding refuses tensors of another element type (a complex128
    waveform would otherwise be read as garbage) and non-contiguous views."""
    c = Cfg("dt", M=2, N=16, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=2)
    ctx = sqngd.Context(c)
    s = torch.ones((1, 2, 16), dtype=torch.complex64, device="cuda")
    with pytest.raises(TypeError):
        ctx.af_forward(s.to(torch.complex128), s)
    with pytest.raises(ValueError):
        ctx.af_forward(s.transpose(1, 2).contiguous().transpose(1, 2), s)
    z = torch.zeros((1, 2, 16), dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        ctx.quantize(z, torch.zeros((1, 8), dtype=torch.float32, device="cuda"))
    ctx.af_forward(s, s)  # the right types pass
    ctx.sync()
