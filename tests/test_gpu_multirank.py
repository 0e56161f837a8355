"""The library's multi-GPU path (include/sqngd.h world > 1) through the C-ABI, on one device.

W contexts of one loopback group (sqngd_create_loopback), each driven by its own host thread and stream,
run exactly the sharded code of world > 1 -- FFT engine: a slice of the (restart, channel, bin) units;
Chebyshev engine: a slice of the (restart, transmit channel) rows -- and the single grouped collective
per evaluation (SUM of the weighted fp64 payload, MAX of the keys, comm.h).  Every rank must return the
full outputs, equal across ranks, matching the fp64 oracle (tests/parity_util.py bars) and the
single-context result.  The loopback reduces in fixed rank order, so the ranks agree bit for bit.
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2604_25728_b200 import configs as CF  # noqa: E402
from paper_2604_25728_b200 import inputs, sqngd  # noqa: E402
from paper_2604_25728_b200.configs import Cfg  # noqa: E402

from parity_util import check_db, check_grad, check_loss, record  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
ENGINES = {"fft": sqngd.ENGINE_FFT, "cheb": sqngd.ENGINE_CHEBYSHEV}
MODES = {"lse": (CF.LOSS_LSE, 60.0), "max": (CF.LOSS_MAX, 0.0), "pnorm": (CF.LOSS_PNORM, 8.0)}


def T(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


def on_ranks(cfg, world, fn, peer=False):
    """fn(ctx, rank) on `world` loopback contexts, one thread + stream each; returns the per-rank results.
    peer: the group reduces with the in-kernel peer-memory all-reduce (k_peer_allreduce) phase by phase."""
    lb = sqngd.Loopback(world, peer=peer)
    ctxs = [sqngd.Context(cfg, loopback=lb, rank=r) for r in range(world)]
    out, errs = [None] * world, []

    def work(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(ctxs[r], r)
                s.synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in ctxs:
        c.close()
    lb.close()
    assert not errs, errs
    assert all(o is not None for o in out), "a rank did not finish"
    return out


def inputs_for(c, seed):
    z = inputs.phase_params(c.R, c.M, c.N, config_index=seed)
    rho = inputs.init_thresholds(c.R, c.B, c.r_n)
    q = O.quantize(c, z, rho)
    w = (q["s_hard"] * np.exp(0.3j * np.cos(0.41 * np.arange(c.N)))).astype(np.complex64)
    return z, rho, q, w


def eval_all(ctx, z, rho, w):
    """Forward metrics, Step-A grad_w and Step-B grad_z / grad_rho of one context."""
    s_h = ctx.quantize(T(z), T(rho))["s_hard"]
    met, p, _ = ctx.af_forward(s_h, T(w))
    mf = ctx.metrics(met)
    met, gw = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_FILTERS)
    mA = ctx.metrics(met)
    met, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
    mB = ctx.metrics(met)
    ctx.sync()
    return dict(mf=mf, p=p.cpu().numpy(), mA=mA, gw=gw.cpu().numpy(), mB=mB, gz=gz.cpu().numpy(), gr=gr.cpu().numpy())


CASES = [
    Cfg("mr-c1", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5, R=2, r_n=4, eps_w=0.4),
    Cfg("mr-ragged", M=3, N=37, B=8, K=21, f_lo=-0.5, f_hi=0.5, R=2, r_n=3),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["lse", "pnorm", "max"])
@pytest.mark.parametrize("engine", ["fft", "cheb"])
@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_sharded_matches_oracle_and_single(c, engine, mode, world):
    lm, bp = MODES[mode]
    c = c.with_(loss_mode=lm, beta_or_p=bp, doppler_engine=ENGINES[engine])
    z, rho, q, w = inputs_for(c, 91)
    res = on_ranks(c, world, lambda ctx, r: eval_all(ctx, z, rho, w))
    single = eval_all(sqngd.Context(c), z, rho, w)
    refF, refp, _ = O.af(c, q["s_hard"], w)
    refA, gw_ref, _ = O.loss_grad(c, q["s_hard"], w, want_s=False)
    refB, _, gs_ref = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs_ref)
    for r in range(world):  # every rank holds the full, identical outputs
        for k in ("gw", "gz", "gr", "p"):
            assert np.array_equal(res[r][k], res[0][k]), (r, k)
        for k in ("mf", "mA", "mB"):  # (snrl_db_max is NaN in the loss+gradient metrics: compare its repr)
            assert repr(res[r][k]) == repr(res[0][k]), (r, k)
    g = res[0]
    for rr in range(c.R):
        check_loss(g["mf"][rr]["loss"], refF[rr]["loss"], "sharded forward loss")
        check_loss(g["mA"][rr]["loss"], refA[rr]["loss"], "sharded Step-A loss")
        check_loss(g["mB"][rr]["loss"], refB[rr]["loss"], "sharded Step-B loss")
        for key in ("wapsl", "wcpsl", "wpsl"):
            check_db(g["mf"][rr][key], refF[rr][key], f"sharded {key}")
        assert g["mf"][rr]["argmax_auto"] == single["mf"][rr]["argmax_auto"]
        assert g["mf"][rr]["argmax_cross"] == single["mf"][rr]["argmax_cross"]
    np.testing.assert_allclose(g["p"], refp, rtol=1e-6, atol=1e-7)
    check_grad(g["gw"], gw_ref, "sharded grad_w")
    check_grad(g["gz"], gz_ref, "sharded grad_z")
    check_grad(g["gr"], gr_ref, "sharded grad_rho")
    d = max(np.linalg.norm(g[k] - single[k]) / np.linalg.norm(single[k]) for k in ("gw", "gz", "gr"))
    record("sharded vs single-context gradient rel", d, 1e-5)
    assert d < 1e-5


@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_sharded_step_matches_single(engine):
    """Three Alg.-1 outer iterations (sqngd_step A+B, eager for the loopback group) on 2 ranks: the state
    stays identical across ranks and within rounding of the single-context run."""
    c = Cfg("mr-step", M=2, N=48, B=4, K=17, f_lo=-0.5, f_hi=0.5, R=2, r_n=4, n_h=2, n_x=2, lr_z=1e-3,
            loss_mode=CF.LOSS_LSE, beta_or_p=60.0, doppler_engine=ENGINES[engine])
    z, rho, q, w0 = inputs_for(c, 93)
    w = q["s_hard"].astype(np.complex64)

    def run(ctx, r):
        st = ctx.new_state(T(z), T(rho), T(w))
        hist = torch.zeros((c.R, c.n_h + c.n_x), dtype=torch.float64, device=DEV)
        for _ in range(3):
            ctx.step(st, sqngd.BLOCK_AB, hist=hist)
        ctx.sync()
        return {k: st[k].cpu().numpy() for k in ("z", "rho", "w")} | {"hist": hist.cpu().numpy()}

    res = on_ranks(c, 2, run)
    single = run(sqngd.Context(c), 0)
    for k in ("z", "rho", "w", "hist"):
        assert np.array_equal(res[1][k], res[0][k]), k
    np.testing.assert_allclose(res[0]["hist"], single["hist"], rtol=1e-6)
    np.testing.assert_allclose(res[0]["w"], single["w"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(res[0]["z"], single["z"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(res[0]["rho"], single["rho"], rtol=0, atol=1e-6)


def test_c5_row_shard_gradient_8_ranks():
    """The Chebyshev engine's row shard at C5 shape (M = 16, N = 4096, P = 8192) with 8 loopback ranks and
    a reduced grid (K = 9 of the C5 grid): the sharded Step-B gradient equals the single-context one."""
    c = CF.C5.with_(R=1, K=9, loss_mode=CF.LOSS_LSE, beta_or_p=200.0, doppler_engine=sqngd.ENGINE_CHEBYSHEV)
    z, rho, q, w = inputs_for(c, 5)

    def run(ctx, r):
        met, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
        m = ctx.metrics(met)
        ctx.sync()
        return m, gz.cpu().numpy(), gr.cpu().numpy()

    res = on_ranks(c, 8, run)
    m1, gz1, gr1 = run(sqngd.Context(c), 0)
    for r in range(8):
        assert np.array_equal(res[r][1], res[0][1]) and np.array_equal(res[r][2], res[0][2])
    check_loss(res[0][0][0]["loss"], m1[0]["loss"], "C5-shape 8-rank loss vs single")
    d = np.linalg.norm(res[0][1] - gz1) / np.linalg.norm(gz1)
    record("C5-shape 8-rank grad_z vs single", d, 1e-5)
    assert d < 1e-5


@pytest.mark.parametrize("mode", ["lse", "pnorm", "max"])
@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_nccl_one_rank_collective_path(engine, mode):
    """The NCCL backend itself on one GPU: an ncclUniqueId with world = 1 runs the sharded code path with
    its grouped collective (k_world_pack, ncclGroupStart / AllReduce SUM fp64 + MAX u64 / GroupEnd,
    k_world_unpack, k_finalize_grad) over a 1-rank communicator; it must match the oracle and the plain
    single-GPU context, eagerly and inside the step's CUDA graph."""
    lm, bp = MODES[mode]
    c = CASES[1].with_(loss_mode=lm, beta_or_p=bp, doppler_engine=ENGINES[engine])
    z, rho, q, w = inputs_for(c, 97)
    ctx = sqngd.Context(c, nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)
    got = eval_all(ctx, z, rho, w)
    single = eval_all(sqngd.Context(c), z, rho, w)
    refA, gw_ref, _ = O.loss_grad(c, q["s_hard"], w, want_s=False)
    refB, _, gs_ref = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs_ref)
    for rr in range(c.R):
        check_loss(got["mA"][rr]["loss"], refA[rr]["loss"], "1-rank NCCL Step-A loss")
        check_loss(got["mB"][rr]["loss"], refB[rr]["loss"], "1-rank NCCL Step-B loss")
        assert got["mf"][rr]["argmax_auto"] == single["mf"][rr]["argmax_auto"]
    check_grad(got["gw"], gw_ref, "1-rank NCCL grad_w")
    check_grad(got["gz"], gz_ref, "1-rank NCCL grad_z")
    check_grad(got["gr"], gr_ref, "1-rank NCCL grad_rho")
    d = max(np.linalg.norm(got[k] - single[k]) / np.linalg.norm(single[k]) for k in ("gw", "gz", "gr"))
    record("1-rank NCCL vs single-context gradient rel", d, 1e-5)
    assert d < 1e-5
    # the step graph with the NCCL calls captured (non-legacy stream), three outer iterations
    cs = c.with_(n_h=2, n_x=2, lr_z=1e-3)
    wq = q["s_hard"].astype(np.complex64)
    res = {}
    for name, kw in (("nccl", dict(nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)), ("single", {})):
        cx = sqngd.Context(cs, **kw)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            st = cx.new_state(T(z), T(rho), T(wq))
            hist = torch.zeros((cs.R, cs.n_h + cs.n_x), dtype=torch.float64, device=DEV)
            for _ in range(3):
                cx.step(st, sqngd.BLOCK_AB, hist=hist)
        s.synchronize()
        cx.sync()
        res[name] = {k: st[k].cpu().numpy() for k in ("z", "rho", "w")} | {"hist": hist.cpu().numpy()}
    np.testing.assert_allclose(res["nccl"]["hist"], res["single"]["hist"], rtol=1e-6)
    np.testing.assert_allclose(res["nccl"]["w"], res["single"]["w"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(res["nccl"]["z"], res["single"]["z"], rtol=0, atol=1e-6)


# ------------------------------------------------- in-kernel all-reduce over peer memory (NEXT-4)
@pytest.mark.parametrize("form", [1, 2], ids=["allreduce", "fused"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["lse", "pnorm", "max"])
@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_peer_allreduce_kernel_in_loopback(engine, mode, world, form):
    """k_peer_allreduce (stage + flag signal, flag wait, rank-ordered read of every rank's stage) as the
    loopback group's reduction, its two phases launched rank by rank (no kernel waits on another): the
    sharded results must equal the plain loopback reduction BIT FOR BIT (both sum in rank order), stay
    identical across ranks, and match the oracle.  Two evaluations per rank and call site use both
    stage parities and growing epochs."""
    lm, bp = MODES[mode]
    c = CASES[1].with_(loss_mode=lm, beta_or_p=bp, doppler_engine=ENGINES[engine])
    z, rho, q, w = inputs_for(c, 95)

    def twice(ctx, r):
        eval_all(ctx, z, rho, w)
        return eval_all(ctx, z, rho, w)

    res = on_ranks(c, world, twice, peer=form)  # 1: k_peer_allreduce between pack and unpack, 2: k_world_peer
    plain = on_ranks(c, world, twice, peer=False)
    for r in range(world):
        for k in ("gw", "gz", "gr", "p"):
            assert np.array_equal(res[r][k], plain[0][k]), (r, k)
        for k in ("mf", "mA", "mB"):
            assert repr(res[r][k]) == repr(plain[0][k]), (r, k)
    _, gw_ref, _ = O.loss_grad(c, q["s_hard"], w, want_s=False)
    _, _, gs_ref = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs_ref)
    check_grad(res[0]["gw"], gw_ref, "peer all-reduce grad_w")
    check_grad(res[0]["gz"], gz_ref, "peer all-reduce grad_z")
    check_grad(res[0]["gr"], gr_ref, "peer all-reduce grad_rho")


@pytest.mark.parametrize("form", [1, 2], ids=["allreduce", "fused"])
def test_peer_allreduce_c5_payload_8_ranks(form):
    """The peer kernel on a payload that spans all its blocks (C5 shape: 1 + 2 M N = 131073 doubles per
    restart, 128 blocks) with 8 ranks: bit-identical to the plain loopback reduction."""
    c = CF.C5.with_(R=1, K=9, loss_mode=CF.LOSS_LSE, beta_or_p=200.0, doppler_engine=sqngd.ENGINE_CHEBYSHEV)
    z, rho, q, w = inputs_for(c, 5)

    def run(ctx, r):
        met, gz, gr = ctx.af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
        m = ctx.metrics(met)
        ctx.sync()
        return m, gz.cpu().numpy(), gr.cpu().numpy()

    res = on_ranks(c, 8, run, peer=form)
    plain = on_ranks(c, 8, run, peer=False)
    for r in range(8):
        assert np.array_equal(res[r][1], plain[0][1]) and np.array_equal(res[r][2], plain[0][2])
        assert repr(res[r][0]) == repr(plain[0][0])


@pytest.mark.parametrize("form", [1, 2], ids=["allreduce", "fused"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_peer_kernels_slices_across_restarts(engine, world, form):
    """R = 3 restarts of 1 + 2 M N = 2401 payload values over 8 blocks of 901: restarts span several blocks
    and blocks straddle two restarts, so the fused kernel's waits on the scalar owners of the touched
    restarts and, for an owner, on the own rank's blocks that still read the local record, all occur.
    Bit-identical to the plain loopback reduction over two evaluations; Step-B gradient vs the oracle."""
    c = Cfg("mr-multi", M=4, N=300, B=4, K=9, f_lo=-0.5, f_hi=0.5, R=3, r_n=4, loss_mode=CF.LOSS_LSE,
            beta_or_p=60.0, doppler_engine=ENGINES[engine])
    z, rho, q, w = inputs_for(c, 99)

    def twice(ctx, r):
        eval_all(ctx, z, rho, w)
        return eval_all(ctx, z, rho, w)

    res = on_ranks(c, world, twice, peer=form)
    plain = on_ranks(c, world, twice, peer=False)
    for r in range(world):
        for k in ("gw", "gz", "gr", "p"):
            assert np.array_equal(res[r][k], plain[0][k]), (r, k)
        for k in ("mf", "mA", "mB"):
            assert repr(res[r][k]) == repr(plain[0][k]), (r, k)
    _, _, gs_ref = O.loss_grad(c, q["s_soft"], w, want_w=False)
    gz_ref, gr_ref = O.chain(c, z, rho, q["s_soft"], gs_ref)
    check_grad(res[0]["gz"], gz_ref, "peer kernels (slices across restarts) grad_z")
    check_grad(res[0]["gr"], gr_ref, "peer kernels (slices across restarts) grad_rho")


MULTI = Cfg("mr-multi1", M=4, N=300, B=4, K=9, f_lo=-0.5, f_hi=0.5, R=3, r_n=4)


@pytest.mark.parametrize("base", [CASES[1], MULTI], ids=lambda c: c.name)
@pytest.mark.parametrize("fused", ["1", "0"], ids=["fused", "allreduce"])
@pytest.mark.parametrize("engine", ["fft", "cheb"])
def test_peer_backend_one_rank_single_launch(engine, fused, base, monkeypatch):
    """The peer backend proper (sqngd_peer_export / sqngd_peer_attach replacing NCCL) at world = 1: the
    single-launch form of the kernel (signal, wait and reduce in one launch, against its own window),
    eagerly and captured in the step's CUDA graph over several replays (the epoch lives in the window,
    so replays need no new arguments).  Must equal the 1-rank NCCL path bit for bit.  mr-multi1 (3 restarts
    over 8 blocks) makes the blocks of one launch wait on one another's flags for real."""
    monkeypatch.setenv("SQNGD_PEER_FUSED", fused)  # read at attach: k_world_peer or pack + k_peer_allreduce + unpack
    c = base.with_(loss_mode=CF.LOSS_LSE, beta_or_p=60.0, doppler_engine=ENGINES[engine])
    z, rho, q, w = inputs_for(c, 97)
    res = {}
    for name in ("peer", "nccl"):
        ctx = sqngd.Context(c, nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)
        if name == "peer":
            ctx.enable_peer_allreduce()
        eval_all(ctx, z, rho, w)
        res[name] = eval_all(ctx, z, rho, w)
        ctx.close()
    for k in ("gw", "gz", "gr", "p"):
        assert np.array_equal(res["peer"][k], res["nccl"][k]), k
    cs = c.with_(n_h=2, n_x=2, lr_z=1e-3)
    wq = q["s_hard"].astype(np.complex64)
    out = {}
    for name in ("peer", "nccl"):
        cx = sqngd.Context(cs, nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)
        if name == "peer":
            cx.enable_peer_allreduce()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            st = cx.new_state(T(z), T(rho), T(wq))
            hist = torch.zeros((cs.R, cs.n_h + cs.n_x), dtype=torch.float64, device=DEV)
            for _ in range(4):
                cx.step(st, sqngd.BLOCK_AB, hist=hist)
        s.synchronize()
        cx.sync()
        out[name] = {k: st[k].cpu().numpy() for k in ("z", "rho", "w")} | {"hist": hist.cpu().numpy()}
        cx.close()
    for k in ("z", "rho", "w", "hist"):
        assert np.array_equal(out["peer"][k], out["nccl"][k]), k


def test_peer_attach_errors():
    """attach before export, and export on a single-GPU context, are rejected (SQNGD_E_INVALID)."""
    import ctypes as C

    c = CASES[0].with_(loss_mode=CF.LOSS_LSE, beta_or_p=60.0)
    plain = sqngd.Context(c)
    buf = C.create_string_buffer(64)
    assert sqngd.lib().sqngd_peer_export(plain.h, buf) == sqngd.E_INVALID
    plain.close()
    ctx = sqngd.Context(c, nccl_uid=sqngd.nccl_unique_id(), rank=0, world=1)
    assert sqngd.lib().sqngd_peer_attach(ctx.h, buf) == sqngd.E_INVALID
    ctx.close()


def test_peer_wait_watchdog_latches_error():
    """A rank that never signals: the waiting kernels give up (2 s in the loopback group), latch the
    time-out bit and return -- sqngd_sync reports SQNGD_E_NCCL on every rank, the GPU does not hang."""
    c = CASES[0].with_(loss_mode=CF.LOSS_LSE, beta_or_p=60.0)
    z, rho, q, w = inputs_for(c, 91)
    lb = sqngd.Loopback(2, peer="drop")
    ctxs = [sqngd.Context(c, loopback=lb, rank=r) for r in range(2)]
    got = [None, None]

    def work(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            try:
                ctxs[r].af_loss_grad(T(z), T(rho), T(w), sqngd.WRT_TRANSMIT)
                ctxs[r].sync()
                got[r] = "no error"
            except sqngd.SqngdError as e:
                got[r] = e.status
            s.synchronize()

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    for cx in ctxs:
        cx.close()
    lb.close()
    assert got == [sqngd.E_NCCL, sqngd.E_NCCL], got
