"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module holds NO arithmetic of the SQNGD method (no quantizer, no AF, no
loss): it only draws numbers.  Both sides of every parity test receive the
*same* fp32 arrays from here; the oracle promotes them exactly to fp64.

Recipe:

* phase parameters  z[r][m][n] = fp32(u),  u = (splitmix64() >> 11) * 2^-53,
  drawn in [r][m][n] order from seed(config, restart) = 1000*config + restart;
  a value that rounds to 1.0f is replaced by nextafterf(1, 0).  This is the
  paper's "random normalized phase Y0" (Alg. 1 Initialization,
  P:L496-499) with the ResNet dropped: z = phi / 2pi in [0, 1).
* thresholds        rho_i = fp32((i + 1/2) / (B r_n)),  i < B r_n
  (uniform midpoints; reproduces Eq. 25's level set).
* filters           w = s_hard(z) (matched-filter start).  That
  needs the hard quantizer, so each side computes it with its own code; this
  module never does.

The paper uses no public dataset or benchmark suite (its inputs are seeded
random phases), so these synthetic inputs *are* the workload.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """`count` successive splitmix64 outputs for the given 64-bit seed."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        x = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * _GOLDEN
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        x = x ^ (x >> np.uint64(31))
    return x


def uniform01_f32(seed: int, count: int) -> np.ndarray:
    """fp32 uniforms in [0, 1) from splitmix64 (53-bit mantissa then fp32 round)."""
    u = (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    f = u.astype(np.float32)
    f[f >= np.float32(1.0)] = np.nextafter(np.float32(1.0), np.float32(0.0))
    return f


def config_seed(config_index: int, restart: int) -> int:
    return 1000 * int(config_index) + int(restart)


def phase_params(R: int, M: int, N: int, config_index: int = 0) -> np.ndarray:
    """z[R][M][N] fp32 in [0,1); restart r uses seed 1000*config_index + r."""
    out = np.empty((R, M, N), dtype=np.float32)
    for r in range(R):
        out[r] = uniform01_f32(config_seed(config_index, r), M * N).reshape(M, N)
    return out


def init_thresholds(R: int, B: int, r_n: int) -> np.ndarray:
    """rho[R][B*r_n] fp32 uniform midpoints (i + 1/2)/(B r_n)."""
    i = np.arange(B * r_n, dtype=np.float64)
    rho = ((i + 0.5) / (B * r_n)).astype(np.float32)
    return np.tile(rho, (R, 1))


def random_unimodular(shape, seed: int) -> np.ndarray:
    """complex64 e^{j 2 pi u}, u uniform -- generic test filters/waveforms."""
    g = np.random.Generator(np.random.PCG64(seed))
    ph = g.random(shape)
    return np.exp(2j * np.pi * ph).astype(np.complex64)


def random_complex(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    """complex64 with iid N(0, scale^2/2) real and imaginary parts."""
    g = np.random.Generator(np.random.PCG64(seed))
    v = g.standard_normal(shape) + 1j * g.standard_normal(shape)
    return (scale * v / np.sqrt(2.0)).astype(np.complex64)


def random_sorted_thresholds(R: int, B: int, r_n: int, seed: int, jitter: float = 0.3) -> np.ndarray:
    """Perturbed (still sorted) thresholds, for tests away from the init grid."""
    g = np.random.Generator(np.random.PCG64(seed))
    n = B * r_n
    i = np.arange(n, dtype=np.float64)
    base = (i + 0.5) / n
    rho = base[None, :] + jitter * (g.random((R, n)) - 0.5) / n
    return np.sort(rho, axis=1).astype(np.float32)


# --------------------------------------------------------------------------- generator (NEXT-2)
# Seeds of the generator draws are offset from the phase-parameter seeds so the streams differ.
_Y0_SEED, _THETA_SEED = 500_000, 700_000


def net_input(R: int, M: int, N: int, B: int, config_index: int = 0) -> np.ndarray:
    """y0[R][M*N] fp32: the random normalized discrete phase Y0 of Alg. 1's initialization
    (Eq. 19 vec() = the [m][n] flattening), levels b/B with b uniform in [0, B)."""
    out = np.empty((R, M * N), dtype=np.float32)
    for r in range(R):
        u = uniform01_f32(_Y0_SEED + config_seed(config_index, r), M * N).astype(np.float64)
        out[r] = (np.floor(u * B) / B).astype(np.float32)
    return out


def net_params(R: int, Din: int, W: int, D: int, config_index: int = 0, bias_scale: float = 0.0) -> np.ndarray:
    """theta[R][P] fp32 in the flat C-ABI layout (include/sqngd.h, sqngd_net_*):
    W_in [W][Din] | b_in [W] | D x (W1 [W][W] | b1 [W] | W2 [W][W] | b2 [W]) | W_out [Din][W] | b_out [Din] | pad
    (pad: zeros up to a multiple of 4 floats).  Weights uniform in +-sqrt(3 / fan_in) (variance 1/fan_in); biases uniform in +-bias_scale
    (0 by default)."""
    sizes = [(W * Din, Din), (W, 0)]
    for _ in range(D):
        sizes += [(W * W, W), (W, 0), (W * W, W), (W, 0)]
    sizes += [(Din * W, W), (Din, 0)]
    P = sum(n for n, _ in sizes)
    out = np.zeros((R, (P + 3) // 4 * 4), dtype=np.float32)  # + pad to the C-ABI's float4 stride
    for r in range(R):
        u = uniform01_f32(_THETA_SEED + config_seed(config_index, r), P).astype(np.float64) * 2.0 - 1.0
        o = 0
        for n, fan_in in sizes:
            scale = np.sqrt(3.0 / fan_in) if fan_in else bias_scale
            out[r, o:o + n] = (u[o:o + n] * scale).astype(np.float32)
            o += n
    return out
