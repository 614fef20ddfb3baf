"""Per-kernel times of the actor forward + backward at a config shape (eager launches, CUDA events
around every launch: spikerl_prof_*). Diagnostic only. Usage:
  python tools/kernel_times.py cfg4 [B] [reps] [--fwd]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
shape, _, B = sg.preset(name)
if len(sys.argv) > 2 and not sys.argv[2].startswith("-"):
    B = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("-") else 5
fwd_only = "--fwd" in sys.argv
torch.cuda.set_device(0)
actor = pk.SpikingActor(pk.actor_cfg_from(shape), B)
actor.load(sg.actor_params(shape, np.random.default_rng(0)))
g = torch.Generator(device="cuda").manual_seed(0)
obs = torch.clamp(torch.randn(B, shape.obs_dim, device="cuda", generator=g), -5, 5)
ga = torch.randn(B, shape.act_dim, device="cuda", generator=g)


def step():
    actor.forward(obs)
    if not fwd_only:
        actor.backward(obs, ga)


step()
torch.cuda.synchronize()
_lib.prof_enable(True)
for _ in range(reps):
    step()
torch.cuda.synchronize()
summ = _lib.prof_summary()
_lib.prof_enable(False)
tot = 0.0
for e in sorted(summ, key=lambda e: -e["total_ms"]):
    ms = e["total_ms"] / reps
    tot += ms
    extra = ""
    if e["bytes"]:
        extra = f"{e['bytes'] / e['launches'] / (e['total_ms'] / e['launches'] / 1e3) / 1e9:8.1f} GB/s"
    if e["flops"]:
        extra = f"{e['flops'] / e['launches'] / (e['total_ms'] / e['launches'] / 1e3) / 1e12:8.1f} TF/s"
    print(f"{e['name']:28s} {ms * 1e3:10.1f} us/step  x{e['launches'] // reps}  {extra}")
print(f"{'sum':28s} {tot * 1e3:10.1f} us/step  ({name}, B={B})")
