"""A "paper-style" comparator on the same GPU: one Step-B loss+gradient
evaluation written the way an autodiff framework runs the paper's method (SQNGD is
"accelerated by GPU" through a framework) -- torch.fft correlations of every (m, l, Doppler bin)
map, a dense |A| tensor, the LSE + SNRL loss (Eqs. 7-10, 37-42 with the LSE surrogate), and
reverse-mode autograd back through the soft quantizer (Eqs. 21-24) to z.

It is measurement context for bench.py only (not the product path, not a parity reference): the
same function as sqngd_af_loss_grad(WRT_TRANSMIT) with LSE, in plain PyTorch ops on the device.
"""
from __future__ import annotations

import math

import torch


class TorchStepB:
    def __init__(self, c, rho, w, device):
        self.c = c
        N, K, M, P = c.N, c.K, c.M, c.P
        self.P = P
        f = torch.linspace(c.f_lo, c.f_hi, K, dtype=torch.float64, device=device) if K > 1 else \
            torch.tensor([c.f_lo], dtype=torch.float64, device=device)
        n1 = torch.arange(1, N + 1, dtype=torch.float64, device=device)
        cyc = torch.remainder(n1[None, :] * f[:, None] / N, 1.0)               # one-based n (Q2)
        self.tw = torch.polar(torch.ones_like(cyc), 2 * math.pi * cyc).to(torch.complex64)  # [K][N]
        self.rho = rho.to(device=device, dtype=torch.float32)                  # [1][B r_n]
        self.w = w.to(device=device, dtype=torch.complex64)                    # [1][M][N]
        wp = torch.zeros((M, P), dtype=torch.complex64, device=device)
        wp[:, :N] = self.w[0]
        self.Hc = torch.conj(torch.fft.fft(wp))                                # [M][P]
        j = torch.arange(P, device=device)
        lag_in = (j < N) | (j > P - N)                                         # tau = -j mod P in [-(N-1), N-1]
        mask = lag_in[None, None, None, :].expand(M, M, 1, P).clone()
        eye = torch.eye(M, dtype=torch.bool, device=device)
        mask[eye[:, :, None, None].expand(M, M, 1, P) & (j == 0)[None, None, None, :]] = False  # auto tau = 0
        self.mask = mask                                                       # [M][M][1][P]
        self.ptar = 10 ** (-c.mu_db / 20)

    def loss_grad(self, z):
        c, N, M, P = self.c, self.c.N, self.c.M, self.P
        z = z.detach().requires_grad_(True)
        a = 1.0 / (2 * c.B)
        y = (a * (torch.tanh(c.c * (z[0][..., None] - self.rho[0])) + 1.0)).sum(-1)   # Q_A (Eq. 24), [M][N]
        s = torch.polar(torch.ones_like(y), 2 * math.pi * y)                            # Eq. 23
        xp = torch.zeros((M, c.K, P), dtype=torch.complex64, device=z.device)
        xp[:, :, :N] = s[:, None, :] * self.tw[None]                                   # Eq. 33
        X = torch.fft.fft(xp)                                                           # [M][K][P]
        r = torch.fft.ifft(X[:, None] * self.Hc[None, :, None, :])                      # Eq. 36, [M][M][K][P]
        v = torch.abs(r) / N                                                            # |A| / N (ifft is 1/P-scaled)
        vs = v.masked_select(self.mask.expand_as(v))
        beta = c.beta_or_p
        l_wpsl = torch.logsumexp(beta * vs, 0) / beta                                   # LSE surrogate of Eq. 37
        p = torch.abs((s * torch.conj(self.w[0])).sum(-1)) / N                          # Eq. 38
        l_snrl = ((p - self.ptar) ** 2).mean()                                          # Eq. 41
        loss = c.eps_w * l_wpsl + (1 - c.eps_w) * l_snrl                                # Eq. 42
        loss.backward()
        return loss.detach(), z.grad


def time_torch_step_b(c, z, rho, w, device, warmup=3, iters=10):
    """(evals/s, ms per eval, loss, dL/dz of the last eval) of the autograd comparator."""
    t = TorchStepB(c, rho, w, device)
    zt = z.to(device)
    for _ in range(warmup):
        t.loss_grad(zt)
    torch.cuda.synchronize(device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        loss, gz = t.loss_grad(zt)
    b.record()
    torch.cuda.synchronize(device)
    ms = a.elapsed_time(b) / iters
    return 1e3 / ms, ms, float(loss), gz
