"""Encoder launch times (eager, events around each launch): the recording forward's enc_fwd against
the inference forward's spikes-only enc_fwd_spikes. Usage: python tools/enc_times.py cfg3L [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3L"
shape, _, B = sg.preset(name)
if len(sys.argv) > 2:
    B = int(sys.argv[2])
actor = pk.SpikingActor(pk.actor_cfg_from(shape), B)
actor.load(sg.actor_params(shape, np.random.default_rng(0)))
obs = torch.clamp(torch.randn(B, shape.obs_dim, device="cuda"), -5, 5)
for rec in (True, False):
    actor.forward(obs, record=rec)
torch.cuda.synchronize()
_lib.prof_enable(True)
for _ in range(10):
    actor.forward(obs, record=True)
    actor.forward(obs, record=False)
torch.cuda.synchronize()
for e in _lib.prof_summary():
    if e["name"].startswith("enc_fwd"):
        print(f"{e['name']:<16s} {e['total_ms'] / e['launches'] * 1e3:8.1f} us/launch  ({name}, B={B})")
_lib.prof_enable(False)
