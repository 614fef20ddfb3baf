"""Second, independent oracle for the surrogate-gradient BPTT: forward-mode dual numbers.

TEST INFRASTRUCTURE ONLY (oracle/__init__.py). Plays the role of SPEC.md:175/649's
"independent tape": the surrogate-relaxed forward graph of oracle/actor.py is re-evaluated
with (value, tangent) pairs, one tangent per parameter, so the directional derivatives of
L = sum(g_a * a) give the whole gradient without any reverse-mode derivation.

Relaxation rules (the definition of the pseudo-gradient; north_star):
  * LIF spike o = [v > V_th] carries tangent h(v) * v_dot with h = z [|v - V_th| < w];
  * reset gate (1 - o_{t-1}): constant (rho = 0) or differentiated (rho = 1);
  * encoder spike o = [acc >= 1]: straight-through, o_dot = acc_dot; soft reset acc -= o
    (so acc_dot becomes acc_dot - o_dot) — DESIGN.md reading R6.
Tiny nets only (P ~ 100 tangents). fp64.
"""
from __future__ import annotations

import numpy as np

F64 = np.float64


class Dual:
    __slots__ = ("v", "d")

    def __init__(self, v, d):
        self.v = np.asarray(v, F64)
        self.d = np.asarray(d, F64)          # shape v.shape + (P,)

    @staticmethod
    def const(v, P):
        v = np.asarray(v, F64)
        return Dual(v, np.zeros(v.shape + (P,)))

    def __add__(self, o):
        if isinstance(o, Dual):
            return Dual(self.v + o.v, self.d + o.d)
        return Dual(self.v + o, self.d)

    __radd__ = __add__

    def __sub__(self, o):
        if isinstance(o, Dual):
            return Dual(self.v - o.v, self.d - o.d)
        return Dual(self.v - o, self.d)

    def __neg__(self):
        return Dual(-self.v, -self.d)

    def __mul__(self, o):
        if isinstance(o, Dual):
            return Dual(self.v * o.v, self.d * o.v[..., None] + o.d * self.v[..., None])
        o = np.asarray(o, F64)
        return Dual(self.v * o, self.d * o[..., None])

    __rmul__ = __mul__

    def __truediv__(self, o):
        if isinstance(o, Dual):
            val = self.v / o.v
            return Dual(val, (self.d - o.d * val[..., None]) / o.v[..., None])
        o = np.asarray(o, F64)
        return Dual(self.v / o, self.d / o[..., None])


def dexp(x: Dual):
    e = np.exp(x.v)
    return Dual(e, x.d * e[..., None])


def dtanh(x: Dual):
    t = np.tanh(x.v)
    return Dual(t, x.d * (1.0 - t * t)[..., None])


def dmatmul_rows(x: Dual, W: Dual):
    """y[b, n] = sum_k x[b, k] W[n, k]."""
    v = x.v @ W.v.T
    d = np.einsum("bkp,nk->bnp", x.d, W.v) + np.einsum("bk,nkp->bnp", x.v, W.d)
    return Dual(v, d)


PARAM_ORDER = ("mu", "sigma", "W1", "W2", "W3", "Wd", "bd")


def _seed_params(p):
    sizes = [np.asarray(p[k]).size for k in PARAM_ORDER]
    P = int(sum(sizes))
    out, off = {}, 0
    for k, n in zip(PARAM_ORDER, sizes):
        val = np.asarray(p[k], F64)
        d = np.zeros(val.shape + (P,))
        d.reshape(n, P)[np.arange(n), off + np.arange(n)] = 1.0
        out[k] = Dual(val, d)
        off += n
    return out, P, sizes


def actor_grads_forward_mode(p, cfg, s, g_a, rho=0.0):
    """Gradient of L = sum(g_a * a) w.r.t. every actor parameter via forward-mode duals."""
    P_, P, sizes = _seed_params(p)
    T, z, w, vth = cfg.T, F64(cfg.surr_height), F64(cfg.surr_window), F64(cfg.v_th)
    s = np.asarray(s, np.float32).astype(F64)
    B, S = s.shape
    E = P_["mu"].v.shape[1]
    # Gaussian receptive fields (dual arithmetic; value re-rounded to fp32 like the encoder)
    diff = Dual.const(s[:, :, None] * np.ones((1, 1, E)), P) - Dual(P_["mu"].v[None], P_["mu"].d[None])
    sg = Dual(P_["sigma"].v[None], P_["sigma"].d[None])
    A = dexp(-((diff * diff) / ((sg * sg) * 2.0)))
    A = Dual(A.v.astype(np.float32).astype(F64).reshape(B, S * E), A.d.reshape(B, S * E, P))
    # encoder spikes, straight-through, soft reset by 1 (fp32 value arithmetic as in R5)
    acc_v = np.zeros((B, S * E), np.float32)
    acc_d = np.zeros((B, S * E, P))
    enc = []
    A32 = A.v.astype(np.float32)
    for t in range(T):
        acc_v = (acc_v + A32).astype(np.float32)
        acc_d = acc_d + A.d
        fire = acc_v >= np.float32(1.0)
        o = Dual(fire.astype(F64), acc_d.copy())     # straight-through
        acc_v = np.where(fire, (acc_v - np.float32(1.0)).astype(np.float32), acc_v)
        acc_d = acc_d - o.d
        enc.append(o)
    x = enc
    for Wname in ("W1", "W2", "W3"):
        W = P_[Wname]
        N = W.v.shape[0]
        c = Dual.const(np.zeros((B, N)), P)
        v = Dual.const(np.zeros((B, N)), P)
        o_prev = Dual.const(np.zeros((B, N)), P)
        outs = []
        for t in range(T):
            c = c * cfg.d_c + dmatmul_rows(x[t], W)
            gate = (Dual.const(np.ones((B, N)), P) - o_prev) if rho else (1.0 - o_prev.v)
            v = (v * cfg.d_v) * gate + c
            h = z * (np.abs(v.v - vth) < w)
            o = Dual((v.v > vth).astype(F64), v.d * h[..., None])
            outs.append(o)
            o_prev = o
        x = outs
    cnt = x[0]
    for t in range(1, T):
        cnt = cnt + x[t]
    fr = cnt / F64(T)
    Wd, bd = P_["Wd"], P_["bd"]
    A_dim, D = Wd.v.shape
    frr = Dual(fr.v.reshape(B, A_dim, D), fr.d.reshape(B, A_dim, D, P))
    prod = frr * Dual(Wd.v[None], Wd.d[None])
    pre = Dual(prod.v.sum(axis=2), prod.d.sum(axis=2)) + Dual(bd.v[None], bd.d[None])
    a = dtanh(pre)
    g_a = np.asarray(g_a, F64)
    Ldot = (a.d * g_a[..., None]).sum(axis=(0, 1))
    out, off = {}, 0
    for k, n in zip(PARAM_ORDER, sizes):
        out[k] = Ldot[off:off + n].reshape(np.asarray(p[k]).shape)
        off += n
    return out, a.v
