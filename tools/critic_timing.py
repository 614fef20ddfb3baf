"""Warm per-call device time of the twin critic through the C ABI (diagnostics): forward only,
forward + update backward (y given), actor-step backward (dQ1/da), at a few batch sizes; CUDA events
around 50 back-to-back calls, then the per-kernel split of one call (spikerl_prof)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk
out = {}
for name, B in (("cfg1", 256), ("cfg2", 512), ("cfg3L", 1024), ("cfg3L", 4096)):
    _, cs, _ = sg.preset(name)
    rng = np.random.default_rng(0)
    c = pk.TwinCritic(pk.critic_cfg(cs.in_dim), B)
    c.load(sg.critic_params(cs, rng), sg.critic_params(cs, rng))
    S = {"cfg1": 17, "cfg2": 111, "cfg3L": 376}[name]
    obs = torch.randn(B, S, device="cuda"); act = torch.rand(B, cs.in_dim - S, device="cuda") * 2 - 1
    y = torch.randn(B, device="cuda")
    res = {}
    ga = torch.zeros(B, cs.in_dim - S, device="cuda")
    for label, kw in (("fwd", {}), ("fwd_bwd", {"y": y}), ("actor_step", {"grad_act": ga, "act_grad_scale": -1.0 / B})):
        for _ in range(5): c(obs, act, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): c(obs, act, **kw)
        e1.record(); torch.cuda.synchronize()
        res[label] = round(e0.elapsed_time(e1) / 50 * 1000, 1)
    from paper_2502_17496_b200 import _lib
    _lib.prof_enable(True)
    c(obs, act, y=y)
    torch.cuda.synchronize()
    res["split_fwd_bwd"] = {e["name"]: round(e["total_ms"] * 1000 / e["launches"], 1) for e in _lib.prof_summary()}
    _lib.prof_enable(False)
    out[f"{name}_B{B}"] = res
print(json.dumps({"us_per_call": out}))
