"""Seeded synthetic inputs shared by the oracle-side tests and the GPU-side tests/bench.

This module holds NO arithmetic of the method: it only draws parameters, observations,
upstream gradients, replay shards and raw noise with numpy's PCG64 (``default_rng``),
with the shapes and distributions BASELINE.json ``configs[0..4]`` prescribe.
Both sides receive the same arrays; neither side imports the other.

Recipe:
  * encoder mu: linspace(-3, 3, E) per obs dim, computed in fp64 then rounded to fp32
    (configs[0] "evenly spaced on [-3,3]"); sigma = 0.15f (configs[0]).
  * W1, W2, W3, Wd and every critic weight ~ U(-sqrt(6/fan_in), +sqrt(6/fan_in))
    ("Kaiming-uniform", configs[0]; reading R13); biases 0.
  * observations ~ N(0,1) clipped to [-5, 5]; upstream action gradient ~ N(0,1).
  * replay: s, s' ~ N(0,1) clipped [-5,5]; a ~ U[-1,1]; r ~ N(0,1); done ~ Bernoulli(0.01).
  * target-policy noise eps ~ N(0, 0.2^2) (raw; the clip to +-0.5 is the method's and is
    applied by each side).
"""
from __future__ import annotations

from dataclasses import dataclass, asdict, replace
import numpy as np


@dataclass(frozen=True)
class ActorShape:
    obs_dim: int          # S
    act_dim: int          # A
    pop_enc: int = 10     # E
    pop_dec: int = 10     # D
    n1: int = 256         # N1
    n2: int = 256         # N2
    T: int = 5
    d_c: float = 0.5
    d_v: float = 0.75
    v_th: float = 0.5
    surr_window: float = 0.5
    surr_height: float = 1.0
    sigma_floor: float = 1e-3
    precision: str = "fp32"   # "fp32" | "bf16"

    @property
    def k0(self) -> int:
        return self.obs_dim * self.pop_enc

    @property
    def n3(self) -> int:
        return self.act_dim * self.pop_dec

    def as_dict(self):
        return asdict(self)


@dataclass(frozen=True)
class CriticShape:
    in_dim: int
    h1: int = 256
    h2: int = 256
    precision: str = "bf16"


@dataclass(frozen=True)
class TD3Hyper:
    gamma: float = 0.99
    tau: float = 0.005
    policy_noise: float = 0.2
    noise_clip: float = 0.5
    policy_delay: int = 2
    lr_actor: float = 1e-4
    lr_critic: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


# BASELINE.json configs[0..4]; "3s"/"3L" are configs[3] at per-rank batch 100 / 4096.
PRESETS = {
    "cfg0": dict(actor=ActorShape(17, 6, precision="fp32"), batch=100),
    "cfg1": dict(actor=ActorShape(17, 6, precision="bf16"), batch=256),
    "cfg2": dict(actor=ActorShape(111, 8, precision="bf16"), batch=512),
    "cfg3s": dict(actor=ActorShape(376, 17, precision="bf16"), batch=100),
    "cfg3L": dict(actor=ActorShape(376, 17, precision="bf16"), batch=4096),
    "cfg4": dict(actor=ActorShape(376, 17, n1=1024, n2=1024, T=16, precision="bf16"), batch=65536),
}


def preset(name: str):
    p = PRESETS[name]
    a = p["actor"]
    return a, CriticShape(a.obs_dim + a.act_dim, precision=a.precision), p["batch"]


def with_(shape, **kw):
    return replace(shape, **kw)


def _he_uniform(rng, fan_out, fan_in):
    bound = np.sqrt(6.0 / fan_in)
    return rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(np.float32)


def actor_params(shape: ActorShape, rng) -> dict:
    S, E, A, D = shape.obs_dim, shape.pop_enc, shape.act_dim, shape.pop_dec
    if E > 1:
        mu_row = np.array([((-3.0) * (E - 1 - e) + 3.0 * e) / (E - 1) for e in range(E)],
                          dtype=np.float64).astype(np.float32)
    else:
        mu_row = np.zeros(1, np.float32)
    return {
        "mu": np.tile(mu_row, (S, 1)).astype(np.float32),
        "sigma": np.full((S, E), 0.15, dtype=np.float32),
        "W1": _he_uniform(rng, shape.n1, shape.k0),
        "W2": _he_uniform(rng, shape.n2, shape.n1),
        "W3": _he_uniform(rng, shape.n3, shape.n2),
        "Wd": _he_uniform(rng, A, D),
        "bd": np.zeros(A, np.float32),
    }


def critic_params(shape: CriticShape, rng) -> dict:
    return {
        "W1": _he_uniform(rng, shape.h1, shape.in_dim), "b1": np.zeros(shape.h1, np.float32),
        "W2": _he_uniform(rng, shape.h2, shape.h1), "b2": np.zeros(shape.h2, np.float32),
        "W3": _he_uniform(rng, 1, shape.h2), "b3": np.zeros(1, np.float32),
    }


def observations(rng, B, S):
    return np.clip(rng.standard_normal((B, S)), -5.0, 5.0).astype(np.float32)


def action_grads(rng, B, A):
    return rng.standard_normal((B, A)).astype(np.float32)


def replay_batch(rng, B, S, A, p_done=0.01):
    return {
        "s": observations(rng, B, S),
        "a": rng.uniform(-1.0, 1.0, size=(B, A)).astype(np.float32),
        "r": rng.standard_normal(B).astype(np.float32),
        "s2": observations(rng, B, S),
        "d": (rng.random(B) < p_done).astype(np.float32),
    }


def target_noise(rng, B, A, std=0.2):
    return (std * rng.standard_normal((B, A))).astype(np.float32)


def randomize_actor(shape: ActorShape, rng, scale=1.0):
    """Tiny-net generator for oracle self-tests: random mu/sigma/weights (not the init recipe)."""
    S, E = shape.obs_dim, shape.pop_enc
    p = actor_params(shape, rng)
    p["mu"] = rng.uniform(-1.0, 1.0, size=(S, E)).astype(np.float32)
    p["sigma"] = rng.uniform(0.3, 1.0, size=(S, E)).astype(np.float32)
    for k in ("W1", "W2", "W3", "Wd"):
        p[k] = (p[k] * scale).astype(np.float32)
    p["bd"] = rng.uniform(-0.2, 0.2, size=shape.act_dim).astype(np.float32)
    return p
