"""Parity protocol helpers.

GPU results come through the C ABI (paper_2502_17496_b200); expected values come only from
oracle/ on the same seeded synthgen inputs.
"""
from __future__ import annotations

import numpy as np

import oracle

NEAR = 1e-5   # north_star: disagreement allowed only within 1e-5 of V_th


def rel_l2(x, ref):
    x = np.asarray(x, np.float64); ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return np.linalg.norm(x - ref) / den if den > 0 else np.linalg.norm(x)


def run_gpu_actor(shape, B, p, s, g_a, engine="auto", reset_grad=0):
    import torch
    import paper_2502_17496_b200 as pk
    actor = pk.SpikingActor(pk.actor_cfg_from(shape, engine=engine, reset_grad=reset_grad), B)
    actor.load(p)
    obs = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    a = actor.forward(obs).cpu().numpy().astype(np.float64)
    grads = None
    if g_a is not None:
        gflat = actor.backward(obs, torch.from_numpy(np.ascontiguousarray(g_a, np.float32)).cuda())
        grads = {k: v.astype(np.float64) for k, v in pk.unpack_actor(actor.cfg, gflat).items()}
    torch.cuda.synchronize()
    tv = actor.tape_view()
    out = dict(a=a, grads=grads, sp=actor.spikes(), A=tv["A"].cpu().numpy(),
               counts=tv["counts"].cpu().numpy())
    return out


def near_fp32_midpoint(a64, ulps=2):
    """True where the fp64 value lies within `ulps` fp64 ulps of a midpoint between two adjacent
    fp32 values: only there may libm's and CUDA's fp64 exp (each within 1 ulp64) round to different
    fp32 results."""
    a64 = np.asarray(a64, np.float64)
    lo = a64.astype(np.float32)
    lo = np.where(lo.astype(np.float64) > a64, np.nextafter(lo, np.float32(-np.inf)), lo)
    hi = np.nextafter(lo, np.float32(np.inf))
    mid = (lo.astype(np.float64) + hi.astype(np.float64)) / 2.0
    return np.abs(a64 - mid) <= ulps * np.spacing(np.abs(a64))


def check_encoder(gpu, shape, p, s, a_stored=True):
    """Stimulation A and encoder spikes bit-exact (north_star). The only exemption is an element whose
    fp64 value sits within 2 ulp64 of an fp32 rounding midpoint; there A may differ by 1 ulp32 and
    that element's column of spikes is compared against the oracle's rule applied to the GPU's A.
    Expected (and observed) exemption count: 0. a_stored=False (a spikes-only forward: no A plane):
    the spikes alone, bit-exact outside such midpoint elements."""
    A_ref = oracle.gaussian_stim(s, p["mu"], p["sigma"])
    O0 = oracle.encode_spikes(A_ref, shape.T)
    if not a_stored:
        mid = near_fp32_midpoint(oracle.gaussian_stim_f64(s, p["mu"], p["sigma"]))
        assert np.array_equal(gpu["sp"]["o0"][:, ~mid], O0[:, ~mid]), "encoder spikes not bit-exact"
        return int(mid.sum())
    diffA = gpu["A"].view(np.uint32).astype(np.int64) - A_ref.view(np.uint32).astype(np.int64)
    bad = diffA != 0
    n_ex = int(bad.sum())
    if n_ex:
        assert np.abs(diffA).max() <= 1, "encoder stimulation differs by more than 1 ulp"
        mid = near_fp32_midpoint(oracle.gaussian_stim_f64(s, p["mu"], p["sigma"]))
        assert np.all(mid[bad]), "encoder stimulation differs away from an fp32 rounding midpoint"
        O0_gpuA = oracle.encode_spikes(gpu["A"], shape.T)
        assert np.array_equal(gpu["sp"]["o0"][:, bad], O0_gpuA[:, bad])
    assert np.array_equal(gpu["sp"]["o0"][:, ~bad], O0[:, ~bad]), "encoder spikes not bit-exact"
    return n_ex


def check_actor(gpu, shape, p, s, g_a, grad_tol=None, act_tol=None, rho=0.0, a_stored=True):
    """Free-running + teacher-forced comparison; returns a stats dict. rho = 1: the reset-gate
    gradient variant (oracle.lif_reverse_scan's rho). a_stored=False: a spikes-only forward (no
    stimulation plane to compare)."""
    prec = shape.precision
    T = shape.T
    sp = gpu["sp"]
    stats = {"enc_exempt": check_encoder(gpu, shape, p, s, a_stored=a_stored)}
    # free-running oracle
    a_free, tape_free = oracle.actor_forward(p, shape, s)
    bad_rows = np.zeros(s.shape[0], bool)
    flips = []
    for l in range(1, 4):
        d = sp[f"o{l}"] != tape_free["O"][l - 1]
        flips.append(int(d.sum()))
        bad_rows |= d.any(axis=(0, 2))
    stats["free_flips"] = flips
    stats["bad_rows"] = int(bad_rows.sum())
    # teacher-forced oracle: every layer driven by the GPU's spikes
    forced = {l: sp[f"o{l}"] for l in range(4)}
    a_tf, tape = oracle.actor_forward(p, shape, s, forced=forced)
    n_spk = 0
    n_exempt = 0
    for l in range(1, 4):
        V = tape["V"][l - 1]
        o_ref = (V > shape.v_th)
        near = np.abs(V - shape.v_th) < NEAR
        mism = (sp[f"o{l}"].astype(bool) != o_ref)
        assert not np.any(mism & ~near), f"layer {l}: spike disagreement away from V_th"
        n_exempt += int((mism & near).sum())
        n_spk += int(o_ref.sum())
        h_ref = np.abs(V - shape.v_th) < shape.surr_window
        near_h = np.minimum(np.abs(V - (shape.v_th - shape.surr_window)),
                            np.abs(V - (shape.v_th + shape.surr_window))) < NEAR
        mh = sp[f"h{l}"].astype(bool) != h_ref
        assert not np.any(mh & ~near_h), f"layer {l}: surrogate-mask disagreement away from the window edge"
    stats["spike_exempt"] = n_exempt
    stats["spikes"] = n_spk
    # north_star: at most 1e-5 of the (oracle's) spikes, strictly (no rounding up to one)
    assert n_exempt <= 1e-5 * n_spk, stats
    # actions: rows without free-running disagreement against the free oracle; all rows against the
    # oracle decoder applied to the GPU's own counts (= a_tf, decoder of forced O3)
    a = gpu["a"]
    if act_tol is None:
        tol = (1e-4 * np.abs(a_tf) + 1e-6) if prec == "fp32" else 2e-2
    else:
        tol = act_tol
    assert np.all(np.abs(a - a_tf) <= tol), ("actions vs decoder(GPU counts)", np.abs(a - a_tf).max())
    good = ~bad_rows
    tolg = tol[good] if np.ndim(tol) else tol
    assert np.all(np.abs(a[good] - a_free[good]) <= tolg), "actions vs free-running oracle"
    stats["max_da"] = float(np.abs(a - a_tf).max())
    # gradients on the GPU's spike tape, masks from the oracle's teacher-forced V
    if g_a is not None and gpu["grads"] is not None:
        ref = oracle.actor_backward(p, shape, tape, g_a, rho=rho)
        gt = grad_tol if grad_tol is not None else (1e-4 if prec == "fp32" else 1e-2)
        errs = {}
        for k in ref:
            e = rel_l2(gpu["grads"][k], ref[k])
            if np.linalg.norm(ref[k]) == 0:
                assert np.linalg.norm(gpu["grads"][k]) <= 1e-6, k
            errs[k] = float(e)
            assert e <= gt, (k, e, gt)
        stats["grad_rel_l2"] = errs
    return stats
