"""TD3 update with the spiking actor — plain CPU oracle.  TEST INFRASTRUCTURE ONLY.

PAPER.md:131 (§III-A "custom implementation of ... TD3"), PAPER.md:135/144 (§IV
average_gradients / DDP allreduce), SPEC.md:235-259 (compute_target, train_step,
soft_update), SPEC.md:278 (Adam), BASELINE.json configs[1] hyper-parameters.
Order per step k (1-based; R15):
  1. a~ = clip(pi'(s') + clip(eps, -c, c), -1, 1)
  2. y = r + gamma (1 - done) min(Q1', Q2')(s', a~)       (no gradient through y)
  3. L_c = mean (Q1 - y)^2 + mean (Q2 - y)^2 ; grads ; allreduce-average ; Adam(critic)
  4. if k % d == 0: L_a = -mean Q1(s, pi(s)) with the critic updated in 3; actor grads;
     allreduce-average; Adam(actor); sigma <- max(sigma, floor); Polyak on actor', Q1', Q2'.
Adam in PyTorch form with its own step counter (R19). fp64 state.
Parity status: pinned (TD3/Adam/Polyak arithmetic pins in tests/test_oracle_pins.py).
"""
from __future__ import annotations

import copy
import numpy as np

from .actor import actor_forward, actor_backward
from .critic import critic_forward, critic_backward

F64 = np.float64


def adam_update(p, g, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """PyTorch Adam (R19): returns (p, m, v) as float64."""
    p = np.asarray(p, F64); g = np.asarray(g, F64)
    m = beta1 * np.asarray(m, F64) + (1.0 - beta1) * g
    v = beta2 * np.asarray(v, F64) + (1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    denom = np.sqrt(v) / np.sqrt(bc2) + eps
    p = p - (lr / bc1) * m / denom
    return p, m, v


def polyak(target, source, tau):
    """theta' <- tau theta + (1 - tau) theta'."""
    return F64(tau) * np.asarray(source, F64) + (1.0 - F64(tau)) * np.asarray(target, F64)


def _f64(d):
    return {k: np.asarray(v, F64) for k, v in d.items()}


def init_state(actor, critic1, critic2):
    z = lambda d: {k: np.zeros_like(np.asarray(v, F64)) for k, v in d.items()}
    return dict(actor=_f64(actor), actor_t=_f64(actor), c=[_f64(critic1), _f64(critic2)],
                c_t=[_f64(critic1), _f64(critic2)], m_a=z(actor), v_a=z(actor),
                m_c=[z(critic1), z(critic2)], v_c=[z(critic1), z(critic2)], t_a=0, t_c=0)


def td3_update(state, acfg, ccfg, hp, batch, eps, k, allreduce=None):
    """One TD3 update; returns (new_state, info). ``allreduce`` averages a flat list of
    gradient dicts across ranks (identity at world = 1)."""
    st = copy.deepcopy(state)
    prec = acfg.precision
    s, a, r, s2, d = (np.asarray(batch[x], F64) for x in ("s", "a", "r", "s2", "d"))
    B = s.shape[0]
    # 1. target policy smoothing
    a2, _ = actor_forward(st["actor_t"], acfg, batch["s2"])
    noise = np.clip(np.asarray(eps, F64), -hp.noise_clip, hp.noise_clip)
    at = np.clip(a2 + noise, -1.0, 1.0)
    # 2. target
    x2 = np.concatenate([s2, at], axis=1)
    q1t, _ = critic_forward(st["c_t"][0], x2, prec)
    q2t, _ = critic_forward(st["c_t"][1], x2, prec)
    y = r + hp.gamma * (1.0 - d) * np.minimum(q1t, q2t)
    # 3. critic loss and update
    x = np.concatenate([s, a], axis=1)
    gc, lc = [], 0.0
    for i in range(2):
        qi, cache = critic_forward(st["c"][i], x, prec)
        lc += np.mean((qi - y) ** 2)
        g, _ = critic_backward(st["c"][i], cache, 2.0 * (qi - y) / B, prec)
        gc.append(g)
    if allreduce is not None:
        gc = allreduce(gc)
    st["t_c"] += 1
    for i in range(2):
        for kname in st["c"][i]:
            st["c"][i][kname], st["m_c"][i][kname], st["v_c"][i][kname] = adam_update(
                st["c"][i][kname], gc[i][kname], st["m_c"][i][kname], st["v_c"][i][kname],
                st["t_c"], hp.lr_critic, hp.beta1, hp.beta2, hp.eps)
    info = dict(critic_loss=lc, y=y, q_target=(q1t, q2t), a_target=at, grads_c=gc)
    # 4. delayed actor + targets
    if k % hp.policy_delay == 0:
        api, tape = actor_forward(st["actor"], acfg, batch["s"])
        xp = np.concatenate([s, api], axis=1)
        q1p, cache = critic_forward(st["c"][0], xp, prec)
        la = -np.mean(q1p)
        _, dx = critic_backward(st["c"][0], cache, np.full(B, -1.0 / B), prec,
                                need_param_grads=False)
        g_a = dx[:, acfg.obs_dim:]
        ga = actor_backward(st["actor"], acfg, tape, g_a)
        if allreduce is not None:
            ga = allreduce([ga])[0]
        st["t_a"] += 1
        for kname in st["actor"]:
            st["actor"][kname], st["m_a"][kname], st["v_a"][kname] = adam_update(
                st["actor"][kname], ga[kname], st["m_a"][kname], st["v_a"][kname],
                st["t_a"], hp.lr_actor, hp.beta1, hp.beta2, hp.eps)
        st["actor"]["sigma"] = np.maximum(st["actor"]["sigma"], F64(acfg.sigma_floor))
        for kname in st["actor"]:
            st["actor_t"][kname] = polyak(st["actor_t"][kname], st["actor"][kname], hp.tau)
        for i in range(2):
            for kname in st["c"][i]:
                st["c_t"][i][kname] = polyak(st["c_t"][i][kname], st["c"][i][kname], hp.tau)
        info.update(actor_loss=la, grads_a=ga, g_a=g_a)
    return st, info
