"""The five BASELINE.json workloads (C1..C5) as plain parameter records.

Readings:
  * Doppler grid: K inclusive uniform bins f_k = f_lo + k (f_hi - f_lo)/(K-1), in
    the paper's units (cycles per CPI, exponent e^{j 2 pi n f / N}).
  * C4 "[-600, 600] in the paper's units": converted to the full unambiguous
    range f in [-N/2, N/2] = [-256, 256] for N = 512 (Q9).
  * r_n = 100, c = 300, eps = 0.1; mu = 0.5 dB.
  * loss surrogate for the dense adjoint: LSE with beta = 200 (Q17).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

LOSS_MAX, LOSS_LSE, LOSS_PNORM = 0, 1, 2


@dataclass(frozen=True)
class Cfg:
    name: str
    M: int
    N: int
    B: int
    K: int
    f_lo: float
    f_hi: float
    R: int = 1
    r_n: int = 100
    c: float = 300.0
    tau_lo: int | None = None      # None -> -(N-1)
    tau_hi: int | None = None      # None -> N-1
    exclude_auto_zero_delay: int = 1
    eps_w: float = 0.1
    mu_db: float = 0.5
    loss_mode: int = LOSS_LSE
    beta_or_p: float = 200.0
    lr_w: float = 5e-2
    lr_z: float = 1e-4
    adam_b1: float = 0.9
    adam_b2: float = 0.999
    adam_eps: float = 1e-8
    n_h: int = 10
    n_x: int = 10
    doppler_engine: int = 0         # 0 auto, 1 per-bin FFT, 2 Chebyshev nodes (include/sqngd.h)
    lr_tol: float = 0.0             # Chebyshev engine error bound (0 => library default 1e-7)
    net_depth: int = 0              # generator residual blocks (paper: 5); 0 with net_width 0
    net_width: int = 0              # generator hidden width (paper: 128); 0 = z is the direct parameter
    lr_theta: float = 1e-5          # Adam rate of the generator parameters (eta_x)
    map_ld: int = 0                 # |A| map row pitch (0 = dense 2N-1; include/sqngd.h)
    iterations: int = 1
    index: int = 0                  # config number used for input seeds

    @property
    def P(self) -> int:
        p = 1
        while p < 2 * self.N - 1:
            p *= 2
        return p

    @property
    def lags(self) -> int:
        return 2 * self.N - 1

    @property
    def BR(self) -> int:
        return self.B * self.r_n

    @property
    def tlo(self) -> int:
        return -(self.N - 1) if self.tau_lo is None else self.tau_lo

    @property
    def thi(self) -> int:
        return (self.N - 1) if self.tau_hi is None else self.tau_hi

    @property
    def cells(self) -> int:
        """Delay-Doppler cells per evaluation per restart: M^2 (2N-1) K."""
        return self.M * self.M * self.lags * self.K

    def with_(self, **kw) -> "Cfg":
        return replace(self, **kw)


C1 = Cfg("C1", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5, iterations=10, index=1)
C2 = Cfg("C2", M=4, N=256, B=8, K=129, f_lo=-0.5, f_hi=0.5, iterations=200, index=2)
C3 = Cfg("C3", M=8, N=1024, B=16, K=257, f_lo=-0.5, f_hi=0.5, iterations=500, index=3)
C4 = Cfg("C4", M=4, N=512, B=8, K=1201, f_lo=-256.0, f_hi=256.0, iterations=300, index=4)
C5 = Cfg("C5", M=16, N=4096, B=16, K=513, f_lo=-0.5, f_hi=0.5, R=8, iterations=50, index=5)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
