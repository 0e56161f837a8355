"""Out-of-bounds write check of the library's kernels (compute-sanitizer is closed on this pool;
DESIGN.md §7 "Hygiene").  With SQNGD_GUARD=1 every workspace buffer of a context is allocated with a
4 KiB guard band on each side (0x5A); after a workload that runs every kernel of the hot path -- both
engines, the three losses, ragged sizes, the |A| map (dense and pitched), Step A / Step B gradients,
graph-replayed sqngd_step with the hard metrics, sqngd_run, the generator, the 2-rank loopback and the
1-rank NCCL collective path -- sqngd_check_guards must report no changed band.  The caller-owned
outputs the test allocates itself (map, gradients) carry guard bands of their own, checked the same way."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
G = 1024  # guard elements around caller-owned outputs


def T(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


@pytest.fixture
def guarded(monkeypatch):
    monkeypatch.setenv("SQNGD_GUARD", "1")
    yield


def padded(shape, dtype):
    """A view of `shape` inside a buffer with G sentinel elements on each side; returns (view, check)."""
    n = int(np.prod(shape))
    real = torch.float32 if dtype == torch.float32 else torch.float32
    per = 2 if dtype == torch.complex64 else 1
    buf = torch.full((n * per + 2 * G,), 1234.5, dtype=real, device=DEV)
    v = buf[G:G + n * per]
    v = (v.view(torch.complex64) if dtype == torch.complex64 else v).view(shape)

    def check():
        torch.cuda.synchronize()
        assert bool((buf[:G] == 1234.5).all()) and bool((buf[G + n * per:] == 1234.5).all()), "caller guard changed"

    return v, check


def workload(c):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=5)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    q = O.quantize(c, z, rho)
    w = (q["s_hard"] * np.exp(0.3j * np.cos(0.41 * np.arange(c.N)))).astype(np.complex64)
    ctx = sqngd.Context(c)
    s_h = ctx.quantize(T(z), T(rho))["s_hard"]
    amap, chk_map = padded((c.R, c.M, c.M, c.K, c.map_ld or 2 * c.N - 1), torch.float32)
    ctx.af_forward(s_h, T(w), map_out=amap)
    gw, chk_gw = padded((c.R, c.M, c.N), torch.complex64)
    ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_FILTERS, outs=(gw,))
    gs, chk_gs = padded((c.R, c.M, c.N), torch.complex64)
    ctx.loss_grad_s(s_h, T(w), sqngd.WRT_TRANSMIT, out=gs)
    ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st = ctx.new_state(T(z), T(rho), T(w))
        hard = torch.empty(c.R * sqngd.METRICS_BYTES, dtype=torch.uint8, device=DEV)
        hist = torch.zeros((c.R, c.n_h + c.n_x), dtype=torch.float64, device=DEV)
        for _ in range(3):
            ctx.step(st, sqngd.BLOCK_AB, hist=hist, hard_met=hard)
        ctx.step(st, sqngd.BLOCK_B, hard_met=hard)
        ctx.run(st, T=3, patience=1)
    s.synchronize()
    ctx.sync()
    for chk in (chk_map, chk_gw, chk_gs):
        chk()
    assert ctx.check_guards() == 0
    ctx.close()


ENGINES = {"fft": sqngd.ENGINE_FFT, "cheb": sqngd.ENGINE_CHEBYSHEV}
MODES = {"lse": (CF.LOSS_LSE, 200.0), "pnorm": (CF.LOSS_PNORM, 16.0), "max": (CF.LOSS_MAX, 0.0)}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("engine", list(ENGINES))
def test_guards_ragged(guarded, engine, mode):
    lm, bp = MODES[mode]
    workload(Cfg("g_rag", M=3, N=37, B=8, K=21, f_lo=-0.5, f_hi=0.5, R=2, r_n=3, n_h=2, n_x=2,
                 loss_mode=lm, beta_or_p=bp, doppler_engine=ENGINES[engine]))


@pytest.mark.parametrize("engine", list(ENGINES))
def test_guards_c2_shape_pitched_map(guarded, engine):
    workload(CF.C2.with_(K=33, n_h=2, n_x=2, map_ld=512, doppler_engine=ENGINES[engine]))


def test_guards_generator(guarded):
    c = CF.C1.with_(net_width=32, net_depth=2, n_h=1, n_x=2, lr_theta=1e-3)
    ctx = sqngd.Context(c)
    th = T(inputs.net_params(1, c.M * c.N, 32, 2, config_index=1))
    y0 = T(inputs.net_input(1, c.M, c.N, c.B, config_index=1))
    zg = ctx.net_forward(th, y0)
    rho = T(inputs.init_thresholds(1, c.B, c.r_n))
    w = ctx.quantize(zg, rho)["s_hard"]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st = ctx.new_state(zg, rho, w, theta=th, y0=y0)
        for _ in range(2):
            ctx.step(st, sqngd.BLOCK_AB)
    s.synchronize()
    ctx.sync()
    assert ctx.check_guards() == 0


def test_guards_collective_paths(guarded):
    import threading

    c = Cfg("g_mr", M=3, N=37, B=8, K=21, f_lo=-0.5, f_hi=0.5, R=2, r_n=3, n_h=2, n_x=2)
    z = inputs.phase_params(c.R, c.M, c.N, config_index=6)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    w = O.quantize(c, z, rho)["s_hard"].astype(np.complex64)
    for eng in ENGINES.values():
        ce = c.with_(doppler_engine=eng)
        lb = sqngd.Loopback(2)
        ctxs = [sqngd.Context(ce, loopback=lb, rank=r) for r in range(2)]

        def work(r):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctxs[r].af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_FILTERS)
                ctxs[r].af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
                s.synchronize()

        th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        for cx in ctxs:
            cx.sync()
            assert cx.check_guards() == 0
            cx.close()
        lb.close()
        one = sqngd.Context(ce, nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)
        one.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
        one.sync()
        assert one.check_guards() == 0
        one.close()


def test_guards_off_reports_minus_one():
    os.environ.pop("SQNGD_GUARD", None)
    ctx = sqngd.Context(Cfg("g_off", M=2, N=16, B=4, K=5, f_lo=-0.5, f_hi=0.5, r_n=2))
    assert ctx.check_guards() == -1
