"""Twin-critic ReLU MLP — plain CPU oracle.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER.md:131 (§III-A "evaluated by the deep critic network ... TD3")
(CriticNet: MLP (state ++ action) -> scalar Q), SPEC.md:279 (2 hidden layers x 256, ReLU);
BASELINE.json configs[1] ("Twin critics are ReLU MLPs 23->256->256->1").
Q = W3 relu(W2 relu(W1 [s;a] + b1) + b2) + b3, input order [s; a], relu'(0) := 0 (R14).
Rounding points in precision="bf16" (R20): the input x, W1..W3, the hidden activations h1,h2
used as GEMM operands, and the activation-gradients dz used as GEMM operands (also for the
bias reduction). Accumulation fp64. Parity status: pinned by central finite differences
(tests/test_oracle_pins.py::test_critic_fd).
"""
from __future__ import annotations

import numpy as np

from .numerics import rounder

F64 = np.float64


def critic_forward(p, x, precision="fp32"):
    q = rounder(precision)
    x0 = q(x)
    z1 = x0 @ q(p["W1"]).T + np.asarray(p["b1"], F64)
    h1 = q(np.maximum(z1, 0.0))
    z2 = h1 @ q(p["W2"]).T + np.asarray(p["b2"], F64)
    h2 = q(np.maximum(z2, 0.0))
    Q = (h2 @ q(p["W3"]).T)[:, 0] + F64(np.asarray(p["b3"]).reshape(-1)[0])
    cache = dict(x0=x0, z1=z1, h1=h1, z2=z2, h2=h2)
    return Q, cache


def critic_backward(p, cache, dQ, precision="fp32", need_param_grads=True):
    """Given dL/dQ [B], return (param grads dict or None, dL/dx [B][in])."""
    q = rounder(precision)
    dQ = np.asarray(dQ, F64)
    W3 = q(p["W3"]); W2 = q(p["W2"]); W1 = q(p["W1"])
    dh2 = dQ[:, None] * W3                               # [B][H2]
    dz2 = q(dh2 * (cache["z2"] > 0))
    dh1 = dz2 @ W2
    dz1 = q(dh1 * (cache["z1"] > 0))
    dx = dz1 @ W1
    g = None
    if need_param_grads:
        g = {
            "W3": (dQ[:, None] * cache["h2"]).sum(axis=0)[None, :],
            "b3": np.array([dQ.sum()]),
            "W2": dz2.T @ cache["h1"], "b2": dz2.sum(axis=0),
            "W1": dz1.T @ cache["x0"], "b1": dz1.sum(axis=0),
        }
    return g, dx
