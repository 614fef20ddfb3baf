"""Timeline of one replay of the configs[4] (or configs[0]) actor step graph — forward + BPTT, as
bench.py captures it — with an event pair around EVERY library launch (spikerl_prof_watch "*").
At this step length the event nodes' few microseconds are noise; the gaps between launches and the
per-kernel intervals are what this shows. Usage: python tools/step_timeline.py [cfg4] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib
import bench

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
shape, _, B = sg.preset(name)
actor = pk.SpikingActor(pk.actor_cfg_from(shape), B)
actor.load(sg.actor_params(shape, np.random.default_rng(0)))
g = torch.Generator(device="cuda").manual_seed(0)
obs = torch.clamp(torch.randn(B, shape.obs_dim, device="cuda", generator=g), -5, 5)
ga = torch.randn(B, shape.act_dim, device="cuda", generator=g)


def step():
    actor.forward(obs)
    actor.backward(obs, ga)


step()
plain_g = bench._capture(step)
w = _lib.Watch("*", 64)
w.arm()
graph = bench._capture(step)
n = w.used()
names = [pk.lib().spikerl_prof_watch_name(i).decode() for i in range(n)]
_lib.Watch.off()
for _ in range(3):
    plain_g.replay()
torch.cuda.synchronize()
plain = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plain_g.replay(); e1.record(); torch.cuda.synchronize()
    plain.append(e0.elapsed_time(e1))
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    t0 = w.ev[0][0]
    rows = sorted((t0.elapsed_time(a), t0.elapsed_time(b), names[i]) for i, (a, b) in enumerate(w.ev[:n]))
    busy = 0.0
    cur_a, cur_b = rows[0][0], rows[0][1]
    for a, b, _ in rows[1:]:
        if a > cur_b:
            busy += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    busy += cur_b - cur_a
    print(f"{name} B={B}: replay {r}: {tot:.3f} ms with {n} watched launches (plain replay median "
          f"{sorted(plain)[len(plain) // 2]:.3f} ms); union of kernel intervals {busy:.3f} ms")
    end = max(x[1] for x in rows)
    prev_end = 0.0
    for a, b, nm in rows:
        bar = " " * int(a / end * 50) + "#" * max(1, int((b - a) / end * 50))
        print(f"  {a:8.3f} {b:8.3f} {b - a:7.3f} gap {a - prev_end:+7.3f}  {nm:<26s} {bar}")
        prev_end = max(prev_end, b)
