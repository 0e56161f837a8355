"""Thin ctypes binding of libsqngd.so (include/sqngd.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch provides
device memory and the current stream.  There is no CPU fallback: if the
extension is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SQNGD_LIB") or os.path.join(_HERE, "libsqngd.so")

OK, E_INVALID, E_DEGENERATE, E_NONFINITE, E_CUDA, E_NCCL, E_NOMEM = range(7)
WRT_FILTERS, WRT_TRANSMIT = 1, 2
BLOCK_A, BLOCK_B, BLOCK_AB = 1, 2, 3
LOSS_MAX, LOSS_LSE, LOSS_PNORM = 0, 1, 2
ENGINE_AUTO, ENGINE_FFT, ENGINE_CHEBYSHEV = 0, 1, 2
FLAG_NO_CROSS, FLAG_TIE, FLAG_DOPPLER_ALIAS = 1, 2, 4  # sqngd_metrics.flags (include/sqngd.h)


class SqngdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sqngd status {status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("R", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("B", C.c_int32), ("r_n", C.c_int32),
        ("c", C.c_double),
        ("K", C.c_int32),
        ("f_lo", C.c_double), ("f_hi", C.c_double),
        ("tau_lo", C.c_int32), ("tau_hi", C.c_int32),
        ("exclude_auto_zero_delay", C.c_int32),
        ("loss_mode", C.c_int32),
        ("beta_or_p", C.c_double),
        ("eps_w", C.c_double),
        ("mu_db", C.c_double),
        ("lr_w", C.c_double), ("lr_z", C.c_double),
        ("adam_b1", C.c_double), ("adam_b2", C.c_double), ("adam_eps", C.c_double),
        ("n_h", C.c_int32), ("n_x", C.c_int32),
        ("weights", C.c_void_p),
        ("doppler_engine", C.c_int32),
        ("lr_tol", C.c_double),
        ("net_depth", C.c_int32), ("net_width", C.c_int32),
        ("lr_theta", C.c_double),
        ("map_ld", C.c_int32),
    ]


class Metrics(C.Structure):
    _fields_ = [
        ("loss", C.c_double), ("loss_wpsl", C.c_double), ("loss_snrl", C.c_double),
        ("wapsl", C.c_double), ("wcpsl", C.c_double), ("wpsl", C.c_double),
        ("argmax_auto", C.c_int32 * 4), ("argmax_cross", C.c_int32 * 4),
        ("flags", C.c_uint32), ("n_cells", C.c_uint32),
        ("apslr_db", C.c_double), ("cpslr_db", C.c_double), ("pslr_db", C.c_double), ("snrl_db_max", C.c_double),
    ]


METRICS_BYTES = C.sizeof(Metrics)


class State(C.Structure):
    _fields_ = [
        ("z", C.c_void_p), ("rho", C.c_void_p), ("w", C.c_void_p),
        ("m_z", C.c_void_p), ("v_z", C.c_void_p), ("m_rho", C.c_void_p), ("v_rho", C.c_void_p),
        ("m_w", C.c_void_p), ("v_w", C.c_void_p),
        ("t_a", C.c_int64), ("t_b", C.c_int64),
        ("theta", C.c_void_p), ("m_theta", C.c_void_p), ("v_theta", C.c_void_p), ("y0", C.c_void_p),
    ]


class RunOpts(C.Structure):
    _fields_ = [("T", C.c_int32), ("patience", C.c_int32), ("check_every", C.c_int32),
                ("require_loss_decrease", C.c_int32), ("tol", C.c_double)]


class RunResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("steps_run", C.c_int64), ("stopped", C.c_int32),
                ("reserved", C.c_int32)]


_lib = None


def lib():
    """Load the in-tree extension; fail loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension {LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
        L.sqngd_create.restype = i32
        L.sqngd_create.argtypes = [C.POINTER(Config), i32, vp, i32, i32, C.POINTER(vp)]
        L.sqngd_destroy.restype = None
        L.sqngd_destroy.argtypes = [vp]
        L.sqngd_last_error.restype = C.c_char_p
        L.sqngd_last_error.argtypes = [vp]
        L.sqngd_sync.restype = i32
        L.sqngd_sync.argtypes = [vp, vp]
        L.sqngd_quantize.restype = i32
        L.sqngd_quantize.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.sqngd_af_forward.restype = i32
        L.sqngd_af_forward.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.sqngd_loss_grad_s.restype = i32
        L.sqngd_loss_grad_s.argtypes = [vp, vp, vp, i32, vp, vp, vp, vp]
        L.sqngd_af_loss_grad.restype = i32
        L.sqngd_af_loss_grad.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]
        L.sqngd_step.restype = i32
        L.sqngd_step.argtypes = [vp, C.POINTER(State), i32, vp, vp, vp]
        L.sqngd_profile_enable.restype = i32
        L.sqngd_profile_enable.argtypes = [vp, i32]
        L.sqngd_check_guards.restype = i32
        L.sqngd_check_guards.argtypes = [vp, C.POINTER(C.c_int64)]
        L.sqngd_profile_read.restype = i32
        L.sqngd_profile_read.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64), i32]
        L.sqngd_num_units.restype = i64
        L.sqngd_num_units.argtypes = [C.POINTER(Config)]
        L.sqngd_shard_range.restype = None
        L.sqngd_shard_range.argtypes = [i64, i32, i32, C.POINTER(i64), C.POINTER(i64)]
        L.sqngd_engine_info.restype = i32
        L.sqngd_engine_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        L.sqngd_net_num_params.restype = i64
        L.sqngd_net_num_params.argtypes = [C.POINTER(Config)]
        L.sqngd_net_forward.restype = i32
        L.sqngd_net_forward.argtypes = [vp, vp, vp, vp, vp]
        L.sqngd_net_backward.restype = i32
        L.sqngd_net_backward.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.sqngd_run.restype = i32
        L.sqngd_run.argtypes = [vp, C.POINTER(State), C.POINTER(RunOpts), C.POINTER(State), vp, vp, vp, vp,
                                C.POINTER(RunResult), vp]
        L.sqngd_loopback_create.restype = vp
        L.sqngd_loopback_create.argtypes = [i32]
        L.sqngd_loopback_destroy.restype = None
        L.sqngd_loopback_destroy.argtypes = [vp]
        L.sqngd_loopback_set_peer.restype = i32
        L.sqngd_loopback_set_peer.argtypes = [vp, i32]
        L.sqngd_peer_export.restype = i32
        L.sqngd_peer_export.argtypes = [vp, vp]
        L.sqngd_peer_attach.restype = i32
        L.sqngd_peer_attach.argtypes = [vp, vp]
        L.sqngd_create_loopback.restype = i32
        L.sqngd_create_loopback.argtypes = [C.POINTER(Config), i32, vp, i32, C.POINTER(vp)]
        L.sqngd_version.restype = C.c_char_p
        L.sqngd_version.argtypes = []
        _lib = L
    return _lib


EXPORTED = ["sqngd_create", "sqngd_destroy", "sqngd_last_error", "sqngd_sync", "sqngd_quantize",
            "sqngd_af_forward", "sqngd_loss_grad_s", "sqngd_af_loss_grad", "sqngd_step",
            "sqngd_profile_enable", "sqngd_profile_read",
            "sqngd_num_units", "sqngd_shard_range", "sqngd_version", "sqngd_engine_info",
            "sqngd_net_num_params", "sqngd_net_forward", "sqngd_net_backward", "sqngd_run",
            "sqngd_loopback_create", "sqngd_loopback_destroy", "sqngd_create_loopback", "sqngd_check_guards",
            "sqngd_loopback_set_peer", "sqngd_peer_export", "sqngd_peer_attach"]


def make_config(cfg, weights_ptr: int | None = None, R: int | None = None) -> Config:
    N = int(cfg.N)
    return Config(
        R=int(cfg.R if R is None else R), M=int(cfg.M), N=N, B=int(cfg.B), r_n=int(cfg.r_n), c=float(cfg.c),
        K=int(cfg.K), f_lo=float(cfg.f_lo), f_hi=float(cfg.f_hi),
        tau_lo=-(N - 1) if getattr(cfg, "tau_lo", None) is None else int(cfg.tau_lo),
        tau_hi=(N - 1) if getattr(cfg, "tau_hi", None) is None else int(cfg.tau_hi),
        exclude_auto_zero_delay=int(getattr(cfg, "exclude_auto_zero_delay", 1)),
        loss_mode=int(getattr(cfg, "loss_mode", LOSS_LSE)), beta_or_p=float(getattr(cfg, "beta_or_p", 200.0)),
        eps_w=float(getattr(cfg, "eps_w", 0.1)), mu_db=float(getattr(cfg, "mu_db", 0.5)),
        lr_w=float(getattr(cfg, "lr_w", 5e-2)), lr_z=float(getattr(cfg, "lr_z", 1e-4)),
        adam_b1=float(getattr(cfg, "adam_b1", 0.9)), adam_b2=float(getattr(cfg, "adam_b2", 0.999)),
        adam_eps=float(getattr(cfg, "adam_eps", 1e-8)),
        n_h=int(getattr(cfg, "n_h", 10)), n_x=int(getattr(cfg, "n_x", 10)),
        weights=weights_ptr,
        doppler_engine=int(getattr(cfg, "doppler_engine", ENGINE_AUTO)),
        lr_tol=float(getattr(cfg, "lr_tol", 0.0)),
        net_depth=int(getattr(cfg, "net_depth", 0)), net_width=int(getattr(cfg, "net_width", 0)),
        lr_theta=float(getattr(cfg, "lr_theta", 1e-5)),
        map_ld=int(getattr(cfg, "map_ld", 0)),
    )


def net_num_params(cfg) -> int:
    """Generator parameters per restart (0 without a generator)."""
    return int(lib().sqngd_net_num_params(C.byref(make_config(cfg))))


def shard_range(units: int, rank: int, world: int) -> tuple[int, int]:
    lo, hi = C.c_int64(), C.c_int64()
    lib().sqngd_shard_range(int(units), int(rank), int(world), C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def metrics_from_bytes(buf: np.ndarray) -> list[dict]:
    """Decode a host copy of an [R] sqngd_metrics device array."""
    raw = np.ascontiguousarray(buf).view(np.uint8)
    n = raw.size // METRICS_BYTES
    out = []
    for r in range(n):
        m = Metrics.from_buffer_copy(raw[r * METRICS_BYTES:(r + 1) * METRICS_BYTES].tobytes())
        d = {k: getattr(m, k) for k, _ in Metrics._fields_}
        d["argmax_auto"] = tuple(m.argmax_auto)
        d["argmax_cross"] = tuple(m.argmax_cross)
        out.append(d)
    return out


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


_DT = {"c64": "complex64", "f32": "float32", "f64": "float64", "u8": "uint8"}


def _tp(t, kind: str) -> int | None:
    """Pointer of a caller tensor the library reads or writes, after checking what the C-ABI assumes:
    a contiguous CUDA tensor of the declared element type (the library takes raw pointers, so a
    complex128 or a non-contiguous view would otherwise be read as garbage)."""
    if t is None:
        return None
    if str(t.dtype).replace("torch.", "") != _DT[kind]:
        raise TypeError(f"sqngd: expected a {_DT[kind]} tensor, got {t.dtype}")
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("sqngd: tensors must be contiguous CUDA tensors")
    return t.data_ptr()


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the same libnccl the library dlopens (torch's bundled NCCL); rank 0
    creates it and every rank passes it to Context(..., nccl_uid=, rank=, world=)."""
    path = "libnccl.so.2"
    try:
        import nvidia.nccl

        for p in nvidia.nccl.__path__:
            cand = os.path.join(p, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                path = cand
                break
    except Exception:
        pass
    L = C.CDLL(path, mode=C.RTLD_GLOBAL)
    buf = C.create_string_buffer(128)
    rc = L.ncclGetUniqueId(buf)
    if rc != 0:
        raise SqngdError(E_NCCL, f"ncclGetUniqueId returned {rc}")
    return buf.raw


class Loopback:
    """Single-device stand-in for NCCL (include/sqngd.h sqngd_loopback_*): `world` contexts of one process,
    each driven by its own host thread, run the library's sharded multi-GPU path."""

    def __init__(self, world: int, peer: bool = False):
        self.world = int(world)
        self.h = lib().sqngd_loopback_create(self.world)
        if not self.h:
            raise SqngdError(E_INVALID, f"sqngd_loopback_create({world})")
        if peer:  # reduce with the peer-memory kernels (phase by phase) instead of the plain reduction:
            # True / 1 = k_peer_allreduce between pack and unpack, 2 / "fused" = k_world_peer (all in one)
            # 3 / "drop": fused, with the last rank's signal phase dropped (the wait watchdog's test)
            st = lib().sqngd_loopback_set_peer(self.h, 3 if peer in (3, "drop") else 2 if peer in (2, "fused") else 1)
            if st != OK:
                raise SqngdError(st, "sqngd_loopback_set_peer")

    def close(self):
        if getattr(self, "h", None):
            lib().sqngd_loopback_destroy(self.h)
            self.h = None


class Context:
    """One library context on one device; tensors are torch CUDA tensors
    (complex64 for s/w/gradients, float32 for z/rho, contiguous)."""

    def __init__(self, cfg, device: int = 0, weights=None, nccl_uid: bytes | None = None, rank: int = 0,
                 world: int = 1, loopback: "Loopback | None" = None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("sqngd needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        self._weights = None
        if weights is not None:
            self._weights = torch.as_tensor(np.asarray(weights, np.float32), device=self.device).contiguous()
        self.R, self.M, self.N, self.B, self.BR = int(cfg.R), int(cfg.M), int(cfg.N), int(cfg.B), int(cfg.B * cfg.r_n)
        self.K, self.L = int(cfg.K), 2 * int(cfg.N) - 1
        self.map_ld = int(getattr(cfg, "map_ld", 0)) or self.L  # |A| map row pitch
        self.c_cfg = make_config(cfg, _ptr(self._weights))
        h = C.c_void_p()
        uid = None
        if nccl_uid is not None:
            uid = C.create_string_buffer(bytes(nccl_uid), 128)
        with torch.cuda.device(self.device):
            if loopback is not None:
                st = lib().sqngd_create_loopback(C.byref(self.c_cfg), device, loopback.h, rank, C.byref(h))
            else:
                st = lib().sqngd_create(C.byref(self.c_cfg), device, uid, rank, world, C.byref(h))
        if st != OK:
            raise SqngdError(st, lib().sqngd_last_error(None).decode())
        self.h = h
        self._met = torch.empty(self.R * METRICS_BYTES, dtype=torch.uint8, device=self.device)

    def enable_peer_allreduce(self, rank: int = 0, world: int = 1):
        """Replace the NCCL backend by the library's own in-kernel all-reduce over peer memory
        (sqngd_peer_export / sqngd_peer_attach): the window handles are exchanged with
        torch.distributed.all_gather_object when world > 1 (argument marshalling only)."""
        mine = C.create_string_buffer(64)
        with self.torch.cuda.device(self.device):
            self._check(lib().sqngd_peer_export(self.h, mine))
            handles = [mine.raw]
            if world > 1:
                import torch.distributed as dist

                handles = [None] * world
                dist.all_gather_object(handles, mine.raw)
            buf = C.create_string_buffer(b"".join(handles), 64 * world)
            self._check(lib().sqngd_peer_attach(self.h, buf))

    def close(self):
        if getattr(self, "h", None):
            lib().sqngd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers
    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def _check(self, st):
        if st != OK:
            raise SqngdError(st, lib().sqngd_last_error(self.h).decode())

    def _c(self, shape):
        return self.torch.empty(shape, dtype=self.torch.complex64, device=self.device)

    def _f(self, shape):
        return self.torch.empty(shape, dtype=self.torch.float32, device=self.device)

    def profile(self, on: bool = True):
        self._check(lib().sqngd_profile_enable(self.h, 1 if on else 0))

    def profile_read(self, reset: bool = True) -> dict:
        ms = (C.c_double * 4)()
        cnt = (C.c_int64 * 4)()
        n = C.c_int64()
        self._check(lib().sqngd_profile_read(self.h, ms, cnt, C.byref(n), 1 if reset else 0))
        return dict(ms=list(ms), count=list(cnt), launches=n.value)

    def engine_info(self) -> dict:
        e, q, err = C.c_int32(), C.c_int32(), C.c_double()
        self._check(lib().sqngd_engine_info(self.h, C.byref(e), C.byref(q), C.byref(err)))
        return {"engine": {ENGINE_FFT: "fft", ENGINE_CHEBYSHEV: "chebyshev"}.get(e.value, "?"), "Q": q.value,
                "err_bound": err.value}

    def sync(self):
        self._check(lib().sqngd_sync(self.h, self._stream()))

    def metrics(self, buf=None) -> list[dict]:
        buf = self._met if buf is None else buf
        return metrics_from_bytes(buf.cpu().numpy())

    # -- entry points
    def quantize(self, z, rho, soft=True, hard=True, want_b=True, want_dq=True) -> dict:
        shp = (self.R, self.M, self.N)
        out = dict(s_soft=self._c(shp) if soft else None, s_hard=self._c(shp) if hard else None,
                   b_hard=self.torch.empty(shp, dtype=self.torch.uint8, device=self.device) if want_b else None,
                   dq=self._f(shp) if want_dq else None)
        self._check(lib().sqngd_quantize(self.h, _tp(z, "f32"), _tp(rho, "f32"), _ptr(out["s_soft"]), _ptr(out["s_hard"]),
                                         _ptr(out["b_hard"]), _ptr(out["dq"]), self._stream()))
        return out

    def af_forward(self, s, w, want_map: bool = False, met_buf=None, want_p: bool = True, snrl_out=None,
                   map_out=None):
        """Forward AF + metrics.  Returns (metrics buffer, p_m [R][M] or None, |A| map or None);
        snrl_out: optional [R][M] float64 tensor that receives SNRL_m (Eq. 10, dB)."""
        amap = map_out if map_out is not None else (self._f((self.R, self.M, self.M, self.K, self.map_ld)) if want_map
                                                    else None)
        p = self.torch.empty((self.R, self.M), dtype=self.torch.float64, device=self.device) if want_p else None
        met = self._met if met_buf is None else met_buf
        self._check(lib().sqngd_af_forward(self.h, _tp(s, "c64"), _tp(w, "c64"), _tp(amap, "f32"), _ptr(met), _tp(p, "f64"), _tp(snrl_out, "f64"),
                                           self._stream()))
        return met, p, amap

    def loss_grad_s(self, s, w, wrt: int, out=None, met_buf=None):
        shp = (self.R, self.M, self.N)
        g = out if out is not None else self._c(shp)
        met = self._met if met_buf is None else met_buf
        gw, gs = (g, None) if wrt == WRT_FILTERS else (None, g)
        self._check(lib().sqngd_loss_grad_s(self.h, _tp(s, "c64"), _tp(w, "c64"), wrt, _ptr(met), _tp(gw, "c64"), _tp(gs, "c64"),
                                            self._stream()))
        return met, g

    def af_loss_grad(self, z, rho, w, wrt: int, outs=None, met_buf=None):
        shp = (self.R, self.M, self.N)
        met = self._met if met_buf is None else met_buf
        if wrt == WRT_FILTERS:
            gw = outs[0] if outs else self._c(shp)
            self._check(lib().sqngd_af_loss_grad(self.h, _tp(z, "f32"), _tp(rho, "f32"), _tp(w, "c64"), wrt, _ptr(met), _tp(gw, "c64"),
                                                 None, None, self._stream()))
            return met, gw
        gz = outs[0] if outs else self._f(shp)
        gr = outs[1] if outs else self._f((self.R, self.BR))
        self._check(lib().sqngd_af_loss_grad(self.h, _tp(z, "f32"), _tp(rho, "f32"), _tp(w, "c64"), wrt, _ptr(met), None,
                                             _tp(gz, "f32"), _tp(gr, "f32"), self._stream()))
        return met, gz, gr

    def net_forward(self, theta, y0, z=None):
        """z = f_theta(y0) ([R][M][N] float32); keeps the tape for net_backward."""
        z = self._f((self.R, self.M, self.N)) if z is None else z
        self._check(lib().sqngd_net_forward(self.h, _ptr(theta), _ptr(y0), _ptr(z), self._stream()))
        return z

    def net_backward(self, theta, y0, z, grad_z, out=None):
        """dL/dtheta [R][P] from grad_z = dL/dz (after net_forward with the same theta, y0)."""
        g = self.torch.empty_like(theta) if out is None else out
        self._check(lib().sqngd_net_backward(self.h, _ptr(theta), _ptr(y0), _ptr(z), _ptr(grad_z), _ptr(g),
                                             self._stream()))
        return g

    def new_state(self, z, rho, w, theta=None, y0=None) -> dict:
        """Optimizer state; with theta [R][P] and y0 [R][M N] (generator mode) z is written by step()."""
        t = self.torch
        st = dict(z=z.clone().contiguous(), rho=rho.clone().contiguous(), w=w.clone().contiguous())
        st["theta"] = st["m_theta"] = st["v_theta"] = st["y0"] = None
        if theta is not None:
            st["theta"] = theta.clone().contiguous()
            st["m_theta"], st["v_theta"] = t.zeros_like(st["theta"]), t.zeros_like(st["theta"])
            st["y0"] = y0.clone().contiguous()
        st["m_z"], st["v_z"] = t.zeros_like(st["z"]), t.zeros_like(st["z"])
        st["m_rho"], st["v_rho"] = t.zeros_like(st["rho"]), t.zeros_like(st["rho"])
        n = st["w"].numel() * 2
        st["m_w"] = t.zeros(n, dtype=t.float32, device=self.device)
        st["v_w"] = t.zeros(n, dtype=t.float32, device=self.device)
        st["t_a"], st["t_b"] = 0, 0
        return st

    def run(self, st: dict, T: int, patience: int, check_every: int = 1, want_hist: bool = True,
            tol: float = 1e-6, require_loss_decrease: bool = True):
        """Alg. 1 driver (sqngd_run): returns (best snapshot dict, best_wpsl [R], best_iter [R],
        wpsl_hist [T][R] or None, result dict with the hard-loss history 'loss_hist'); `st` is
        advanced in place."""
        t = self.torch
        best = {k: t.empty_like(st[k]) for k in ("z", "rho", "w")}
        best["theta"] = t.empty_like(st["theta"]) if st.get("theta") is not None else None
        bw = t.empty(self.R, dtype=t.float64, device=self.device)
        bi = t.empty(self.R, dtype=t.int32, device=self.device)
        hist = t.full((T, self.R), float("nan"), dtype=t.float64, device=self.device) if want_hist else None
        lhist = t.full((T, self.R), float("nan"), dtype=t.float64, device=self.device) if want_hist else None
        cs = self._cstate(st)
        cb = State(z=_ptr(best["z"]), rho=_ptr(best["rho"]), w=_ptr(best["w"]), theta=_ptr(best["theta"]))
        res = RunResult()
        opts = RunOpts(T=int(T), patience=int(patience), check_every=int(check_every),
                       require_loss_decrease=1 if require_loss_decrease else 0, tol=float(tol))
        self._check(lib().sqngd_run(self.h, C.byref(cs), C.byref(opts), C.byref(cb), _ptr(bw), _ptr(bi), _ptr(hist),
                                    _ptr(lhist), C.byref(res), self._stream()))
        st["t_a"], st["t_b"] = cs.t_a, cs.t_b
        return best, bw, bi, hist, {"iterations": res.iterations, "steps_run": res.steps_run,
                                    "stopped": bool(res.stopped), "loss_hist": lhist}

    def _cstate(self, st: dict) -> State:
        return State(z=_ptr(st["z"]), rho=_ptr(st["rho"]), w=_ptr(st["w"]), m_z=_ptr(st["m_z"]), v_z=_ptr(st["v_z"]),
                     m_rho=_ptr(st["m_rho"]), v_rho=_ptr(st["v_rho"]), m_w=_ptr(st["m_w"]), v_w=_ptr(st["v_w"]),
                     t_a=int(st["t_a"]), t_b=int(st["t_b"]),
                     theta=_ptr(st.get("theta")), m_theta=_ptr(st.get("m_theta")),
                     v_theta=_ptr(st.get("v_theta")), y0=_ptr(st.get("y0")))

    def check_guards(self) -> int:
        """Buffers whose guard bands changed (SQNGD_GUARD=1 at create), or -1 without guards."""
        n = C.c_int64(0)
        self._check(lib().sqngd_check_guards(self.h, C.byref(n)))
        return int(n.value)

    def step(self, st: dict, block: int = BLOCK_AB, hist=None, hard_met=None):
        cs = State(z=_tp(st["z"], "f32"), rho=_tp(st["rho"], "f32"), w=_tp(st["w"], "c64"),
                   m_z=_tp(st["m_z"], "f32"), v_z=_tp(st["v_z"], "f32"), m_rho=_tp(st["m_rho"], "f32"),
                   v_rho=_tp(st["v_rho"], "f32"), m_w=_ptr(st["m_w"]), v_w=_ptr(st["v_w"]),
                   t_a=int(st["t_a"]), t_b=int(st["t_b"]),
                   theta=_tp(st.get("theta"), "f32"), m_theta=_tp(st.get("m_theta"), "f32"),
                   v_theta=_tp(st.get("v_theta"), "f32"), y0=_tp(st.get("y0"), "f32"))
        self._check(lib().sqngd_step(self.h, C.byref(cs), int(block), _ptr(hist), _ptr(hard_met), self._stream()))
        st["t_a"], st["t_b"] = cs.t_a, cs.t_b
        return st
