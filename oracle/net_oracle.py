"""fp64 numpy oracle of the transmit-side generator z = f_theta(y0) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may import
this module.  It shares no code with the CUDA path (paper_2604_25728_b200/csrc/net*.cu).

What it follows:
  * PAPER.md Eq. 20: "A deep residual network (ResNet) is employed to generate
    continuous phase variables z = f_theta(y0)", y0 = vec(Y0) (Eq. 19), Y0 the
    random normalized discrete phase of Alg. 1's initialization.
  * "5 residual blocks and a hidden width of 128, ... hidden and residual layers
    mainly use the tanh activation function, and a sigmoid activation is adopted at the output".
  * Readings (DESIGN.md §3 "Generator"; SPEC.md generator-net S:L348-407 for the block shape):
        h_0     = tanh(W_in y0 + b_in)                               input layer, width W
        u_d     = tanh(W1_d h_d + b1_d)                              d = 0 .. D-1
        h_{d+1} = h_d + W2_d u_d + b2_d                              residual skip around both
        z       = sigmoid(W_out h_D + b_out)                          z in (0, 1)^{M N}
  * Flat parameter layout theta (the C-ABI's, include/sqngd.h):
        W_in [W][Din] | b_in [W] | D x (W1 [W][W] | b1 [W] | W2 [W][W] | b2 [W]) | W_out [Din][W] | b_out [Din]
    count = 2 W Din + W + D (2 W^2 + 2 W) + Din.

Reverse mode is written out layer by layer (the chain rule of the forward above, in reverse
order); the tests pin it by central finite differences, not by re-deriving it.
"""
from __future__ import annotations

import numpy as np


def num_params(Din: int, W: int, D: int) -> int:
    return 2 * W * Din + W + D * (2 * W * W + 2 * W) + Din


def unpack(theta: np.ndarray, Din: int, W: int, D: int) -> dict:
    """Views into the flat parameter vector (same memory).  Entries past num_params (the C-ABI's
    float4 stride padding, < 4 floats) are ignored."""
    theta = np.asarray(theta)
    n = num_params(Din, W, D)
    assert theta.ndim == 1 and n <= theta.size < n + 4, theta.shape
    theta = theta[:n]
    o = 0

    def take(n, shape):
        nonlocal o
        v = theta[o:o + n].reshape(shape)
        o += n
        return v

    p = {"W_in": take(W * Din, (W, Din)), "b_in": take(W, (W,)), "blocks": []}
    for _ in range(D):
        p["blocks"].append({"W1": take(W * W, (W, W)), "b1": take(W, (W,)),
                            "W2": take(W * W, (W, W)), "b2": take(W, (W,))})
    p["W_out"] = take(Din * W, (Din, W))
    p["b_out"] = take(Din, (Din,))
    assert o == n
    return p


def forward(theta, y0, Din: int, W: int, D: int):
    """z = f_theta(y0) in fp64 and the tape {h: [h_0..h_D], u: [u_0..u_{D-1}], z}."""
    th = np.asarray(theta, np.float64)
    y0 = np.asarray(y0, np.float64).reshape(Din)
    p = unpack(th, Din, W, D)
    h = np.tanh(p["W_in"] @ y0 + p["b_in"])
    hs, us = [h], []
    for b in p["blocks"]:
        u = np.tanh(b["W1"] @ h + b["b1"])
        h = h + b["W2"] @ u + b["b2"]
        us.append(u)
        hs.append(h)
    o = p["W_out"] @ h + p["b_out"]
    z = 1.0 / (1.0 + np.exp(-o))
    return z, {"h": hs, "u": us, "z": z, "y0": y0}


def backward(theta, tape: dict, gz, Din: int, W: int, D: int):
    """dL/dtheta (flat, same layout and length as theta; 0 in any padding) and dL/dy0 for the
    upstream dL/dz."""
    th = np.asarray(theta, np.float64)
    p = unpack(th, Din, W, D)
    g = np.zeros_like(th)
    gp = unpack(g, Din, W, D)
    gz = np.asarray(gz, np.float64).reshape(Din)
    z, hs, us, y0 = tape["z"], tape["h"], tape["u"], tape["y0"]
    go = gz * z * (1.0 - z)                       # sigmoid'
    gp["W_out"][...] = np.outer(go, hs[D])
    gp["b_out"][...] = go
    gh = p["W_out"].T @ go
    for d in range(D - 1, -1, -1):
        b, gb = p["blocks"][d], gp["blocks"][d]
        u, h = us[d], hs[d]
        gb["W2"][...] = np.outer(gh, u)
        gb["b2"][...] = gh
        ga = (b["W2"].T @ gh) * (1.0 - u * u)     # tanh'
        gb["W1"][...] = np.outer(ga, h)
        gb["b1"][...] = ga
        gh = gh + b["W1"].T @ ga                  # skip path + inner path
    ga0 = gh * (1.0 - hs[0] * hs[0])
    gp["W_in"][...] = np.outer(ga0, y0)
    gp["b_in"][...] = ga0
    gy0 = p["W_in"].T @ ga0
    return g, gy0


def forward_batch(theta, y0, Din, W, D):
    """[R][P] parameters, [R][Din] inputs -> z [R][Din] and the per-restart tapes."""
    out, tapes = [], []
    for r in range(theta.shape[0]):
        z, t = forward(theta[r], y0[r], Din, W, D)
        out.append(z)
        tapes.append(t)
    return np.stack(out), tapes


def backward_batch(theta, tapes, gz, Din, W, D):
    return np.stack([backward(theta[r], tapes[r], gz[r].reshape(Din), Din, W, D)[0]
                     for r in range(theta.shape[0])])
