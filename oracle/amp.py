"""Dynamic loss scaling (GradScaler) state machine — plain CPU oracle.  TEST INFRASTRUCTURE ONLY.

PAPER.md:164-167 (§IV-A: "the GradScaler ... scales the loss function during the backward pass to
maintain gradient magnitude, adjusting the scale as necessary to prevent overflow"). The rule is
PyTorch's torch.cuda.amp.GradScaler, which the paper names:
  - the loss (here: its gradient dL/dQ) is multiplied by the scale S before the backward;
  - before the optimizer step the gradients are checked: any inf / NaN -> the step is skipped
    (parameters, moments and the optimizer's step count unchanged); else they are multiplied by
    1/S and the step runs;
  - update: on a skipped step S <- S * backoff and the finite-step count resets; otherwise the
    count increments and, when it reaches growth_interval, S <- S * growth and the count resets.
Parity status: pinned (hand-worked sequences in tests/test_oracle_pins.py).
"""
from __future__ import annotations

import numpy as np


def amp_step(state, grads_finite: bool, growth=2.0, backoff=0.5, interval=2000):
    """One optimizer step of the scaler. state = (scale, count); returns (new_state, step_taken)."""
    scale, count = state
    if not grads_finite:
        return (scale * backoff, 0), False
    count += 1
    if count == interval:
        return (scale * growth, 0), True
    return (scale, count), True


def unscale(g, scale):
    """g * (1 / S) in fp32 (PyTorch multiplies by the fp32 reciprocal of the scale)."""
    inv = np.float32(1.0) / np.float32(scale)
    return (np.asarray(g, np.float32) * inv).astype(np.float32)


def all_finite(g) -> bool:
    return bool(np.all(np.isfinite(np.asarray(g))))
