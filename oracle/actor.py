"""Population-coded spiking actor (PopSAN-style) — plain CPU oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module.

Follows, step by step and in the paper's order:
  PAPER.md:129-131 (§III-A "DeepRL-SNN with Population Encoding and Decoding"): Gaussian
    population encoding of each observation dimension -> spike trains -> multi-layer fully
    connected LIF SNN ("integrates presynaptic spikes into a current, which then charges the
    membrane voltage ... fires") -> firing rates -> weighted sum -> actions.
  BASELINE.json north_star: deterministic soft-reset encoder spikes; current-based LIF
    c = d_c*c + W*o, v = d_v*v*(1-o_prev) + c, o = [v > V_th]; rectangular pseudo-gradient BPTT.
  SPEC.md:123-176 (snn-actor ops gaussian_stim, encode_spikes, lif_step, decode_action,
    actor_forward, actor_backward) for interfaces and examples.
Every reading where the sources are silent is listed in DESIGN.md "Readings" (R1..R30) and
cited below by number.

Precision: fp64 everywhere except (i) the encoder rule, which is fp32 by definition (R4, R5),
and (ii) in precision="bf16" the GEMM operands named in R20 are rounded to bf16 (fp64
accumulation of the rounded operands).

Array layout: every per-timestep array is [T][B][N] (t-major).
Parity status: pinned (tests/test_oracle_pins.py: hand traces, golden tiny net, T=1 closed
form, zero-weight cases, forward-mode dual-number second oracle, finite differences).
"""
from __future__ import annotations

import numpy as np

from .numerics import rounder

F64 = np.float64


# ----------------------------------------------------------------------------- forward
def gaussian_stim(s, mu, sigma):
    """A[b, i*E+e] = RNE_fp32(exp(-(s_bi - mu_ie)^2 / (2 sigma_ie^2))).

    PAPER.md:131 ("populations use Gaussian distributions to transform continuous input
    values"); SPEC.md:123-131 gaussian_stim. fp64 evaluation of the exponent from the fp32
    inputs with the op sequence d=s-mu; q=d*d; den=2*(sigma*sigma); exp(-(q/den)) (R4),
    then one rounding to fp32. Flattening k = i*E + e (R1).
    """
    return gaussian_stim_f64(s, mu, sigma).astype(np.float32)


def gaussian_stim_f64(s, mu, sigma):
    """The fp64 value gaussian_stim rounds to fp32 (same op sequence, R4), [B][S*E]; the parity
    protocol's encoder exemption (C-4 step 2) is decided on it."""
    s64 = np.asarray(s, np.float32).astype(F64)
    mu64 = np.asarray(mu, np.float32).astype(F64)
    sg64 = np.asarray(sigma, np.float32).astype(F64)
    if np.any(sg64 <= 0):
        raise ValueError("sigma must be > 0 (SPEC.md:127)")
    d = s64[:, :, None] - mu64[None, :, :]
    q = d * d
    den = 2.0 * (sg64 * sg64)
    A = np.exp(-(q / den[None, :, :]))
    return A.reshape(s64.shape[0], -1)


def encode_spikes(A, T):
    """Deterministic soft-reset accumulate-and-fire encoder (north_star).

    fp32 accumulator: acc += A; spike iff acc >= 1.0f; then acc -= 1.0f (R5: '>=' is what
    SPEC.md:138,140's examples require). Returns uint8 [T][B][K0].
    """
    A = np.asarray(A, np.float32)
    acc = np.zeros_like(A, dtype=np.float32)
    one = np.float32(1.0)
    out = np.zeros((T,) + A.shape, dtype=np.uint8)
    for t in range(T):
        acc = (acc + A).astype(np.float32)
        fire = acc >= one
        out[t] = fire
        acc = np.where(fire, (acc - one).astype(np.float32), acc).astype(np.float32)
    return out


def lif_layer_forward(o_in, W, d_c, d_v, v_th, forced_o=None):
    """Current-based LIF layer over T steps (north_star equations).

    For t = 1..T:  I_t = W o_in_t;  c_t = d_c c_{t-1} + I_t;
                   v_t = d_v v_{t-1} (1 - o_{t-1}) + c_t;  o_t = [v_t > V_th].
    Zero initial state, no bias, same-step propagation (R7). fp64.
    ``forced_o`` (teacher forcing, DESIGN.md parity protocol): if given, the reset gate of
    step t+1 uses forced_o[t] instead of this layer's own decision.
    Returns (V [T][B][N] float64, O [T][B][N] uint8, I [T][B][N] float64).
    """
    o_in = np.asarray(o_in)
    T, B, _ = o_in.shape
    W = np.asarray(W, F64)
    N = W.shape[0]
    d_c, d_v, v_th = F64(d_c), F64(d_v), F64(v_th)
    c = np.zeros((B, N), F64)
    v = np.zeros((B, N), F64)
    o_prev = np.zeros((B, N), F64)
    V = np.empty((T, B, N), F64)
    O = np.empty((T, B, N), np.uint8)
    Ic = np.empty((T, B, N), F64)
    for t in range(T):
        I = o_in[t].astype(F64) @ W.T
        c = d_c * c + I
        v = d_v * v * (1.0 - o_prev) + c
        o = v > v_th
        V[t], O[t], Ic[t] = v, o, I
        o_prev = (forced_o[t] if forced_o is not None else o).astype(F64)
    return V, O, Ic


def decode(O3, Wd, bd, T):
    """Firing-rate decoder ("aggregates these spikes over time to compute firing
    rates, which are then translated into real-valued actions through a weighted sum";
    SPEC.md:150-158).  cnt = sum_t o; fr = cnt/T; a_j = tanh(sum_d Wd[j,d] fr[j*D+d] + bd_j)
    with action-major flattening n = j*D + d (R1) and bound 1 (R9)."""
    Wd = np.asarray(Wd, F64)
    A, D = Wd.shape
    cnt = np.asarray(O3).astype(F64).sum(axis=0)          # [B][N3]
    fr = cnt / F64(T)
    pre = (fr.reshape(-1, A, D) * Wd[None]).sum(axis=-1) + np.asarray(bd, F64)[None]
    return np.tanh(pre), fr, pre


def actor_forward(p, cfg, s, forced=None):
    """Encoder -> 3 LIF layers -> decoder. Returns (a, tape).

    ``forced``: optional dict {0: enc spikes, 1: O1, 2: O2, 3: O3} of externally supplied
    spike trains ([T][B][N] 0/1). When layer l is forced, the *forced* spikes are used both for
    the layer's reset gate and as the next layer's input, while V_l is still computed by the
    oracle (teacher forcing).
    """
    q = rounder(cfg.precision)
    T = cfg.T
    A = gaussian_stim(s, p["mu"], p["sigma"])
    O0_own = encode_spikes(A, T)
    O0 = O0_own if not forced or 0 not in forced else np.asarray(forced[0], np.uint8)
    o_in = O0
    Ws = [q(p["W1"]), q(p["W2"]), q(p["W3"])]
    V, O, I = [], [], []
    for l in range(3):
        fo = None if not forced or (l + 1) not in forced else np.asarray(forced[l + 1], np.uint8)
        v_l, o_l, i_l = lif_layer_forward(o_in, Ws[l], cfg.d_c, cfg.d_v, cfg.v_th, forced_o=fo)
        V.append(v_l); I.append(i_l)
        o_used = o_l if fo is None else fo
        O.append(o_used)
        o_in = o_used
    a, fr, pre = decode(O[2], p["Wd"], p["bd"], T)
    tape = dict(A=A, O0=O0, O0_own=O0_own, O=O, V=V, I=I, a=a, fr=fr, pre=pre,
                s=np.asarray(s, np.float32))
    return a, tape


# ---------------------------------------------------------------------------- backward
def surrogate(V, v_th, w, z):
    """Rectangular pseudo-gradient h(v) = z * [|v - V_th| < w] (configs[0] "rectangular
    pseudo-gradient with window 0.5"; strict '<' and z = 1 by default, R10)."""
    return F64(z) * (np.abs(np.asarray(V, F64) - F64(v_th)) < F64(w))


def lif_reverse_scan(g_o, V, O, d_c, d_v, v_th, w, z, rho=0.0, H=None):
    """BPTT through one LIF layer (DESIGN.md derivation R11).

    With delta_v_{T+1} = delta_c_{T+1} = 0, for t = T..1:
        delta_v_t = h_t (g_o_t - rho d_v v_t delta_v_{t+1}) + d_v (1 - o_t) delta_v_{t+1}
        delta_c_t = delta_v_t + d_c delta_c_{t+1}
        G_t = delta_c_t   (= dL/dI_t)
    rho = 0: reset gate (1 - o_{t-1}) detached (default); rho = 1: through it.
    ``H`` optionally supplies the surrogate values (e.g. masks recomputed elsewhere).
    """
    T = V.shape[0]
    d_c, d_v = F64(d_c), F64(d_v)
    if H is None:
        H = surrogate(V, v_th, w, z)
    dv_next = np.zeros(V.shape[1:], F64)
    dc_next = np.zeros(V.shape[1:], F64)
    G = np.empty(V.shape, F64)
    for t in range(T - 1, -1, -1):
        h = H[t]
        dv_t = h * (g_o[t] - F64(rho) * d_v * V[t] * dv_next) + d_v * (1.0 - O[t].astype(F64)) * dv_next
        dc_t = dv_t + d_c * dc_next
        G[t] = dc_t
        dv_next, dc_next = dv_t, dc_t
    return G


def actor_backward(p, cfg, tape, g_a, rho=0.0, masks=None):
    """Reverse mode through decoder, 3 LIF layers and the encoder.

    g_a = dL/da [B][A] (used directly, R25). Rounding points in precision="bf16" (R20): W_l
    operands, G_l before the dX/dW contractions, and sum_t G_1 before the encoder contraction.
    ``masks``: optional list of 3 surrogate arrays [T][B][N_l] overriding h computed from V.
    Returns dict of fp64 gradients with the parameter names of actor_params().
    """
    q = rounder(cfg.precision)
    T = cfg.T
    a = tape["a"]; fr = tape["fr"]
    Wd = np.asarray(p["Wd"], F64)
    A_dim, D = Wd.shape
    g_a = np.asarray(g_a, F64)
    # decoder (fp32-class: never rounded, R20)
    g_pre = g_a * (1.0 - a * a)                                    # [B][A]
    dbd = g_pre.sum(axis=0)
    dWd = (g_pre[:, :, None] * fr.reshape(-1, A_dim, D)).sum(axis=0)
    g_fr = (g_pre[:, :, None] * Wd[None]).reshape(-1, A_dim * D)  # [B][N3]
    g_o = np.broadcast_to(g_fr / F64(T), (T,) + g_fr.shape).copy()  # constant in t (C-1 step 2)
    Ws = [q(p["W1"]), q(p["W2"]), q(p["W3"])]
    O_in = [tape["O0"], tape["O"][0], tape["O"][1]]
    grads = {}
    Gsum1 = None
    for l in (2, 1, 0):
        H = None if masks is None else np.asarray(masks[l], F64)
        G = lif_reverse_scan(g_o, tape["V"][l], tape["O"][l], cfg.d_c, cfg.d_v, cfg.v_th,
                             cfg.surr_window, cfg.surr_height, rho=rho, H=H)
        if l == 0:
            Gsum1 = q(G.sum(axis=0))                               # sum_t G1, then rounded
        Gq = q(G)
        o_prev = O_in[l].astype(F64)
        grads[f"W{l+1}"] = np.einsum("tbn,tbk->nk", Gq, o_prev)
        if l > 0:
            g_o = np.einsum("tbn,nk->tbk", Gq, Ws[l])
    # encoder: dL/dA = (sum_t G1) W1 (straight-through spikes with reset-by-1: do_t/dA = 1)
    gA = Gsum1 @ Ws[0]                                             # [B][K0]
    s = tape["s"].astype(F64)
    mu = np.asarray(p["mu"], np.float32).astype(F64)
    sg = np.asarray(p["sigma"], np.float32).astype(F64)
    S, E = mu.shape
    Aval = tape["A"].astype(F64).reshape(-1, S, E)
    gA = gA.reshape(-1, S, E)
    d = s[:, :, None] - mu[None]
    grads["mu"] = (gA * Aval * d / (sg * sg)[None]).sum(axis=0)
    grads["sigma"] = (gA * Aval * d * d / (sg * sg * sg)[None]).sum(axis=0)
    grads["Wd"] = dWd
    grads["bd"] = dbd
    return grads


def counts(tape):
    return tape["O"][2].astype(np.int64).sum(axis=0)
