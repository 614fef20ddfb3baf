"""Timeline of one replay of a TD3 update-pair graph with an event pair around EVERY library launch
(spikerl_prof_watch "*", recorded as graph event nodes). The event nodes are far from free: each cuts
the programmatic-launch overlap at its boundary and costs a few microseconds, so the absolute times
are inflated ~2x at configs[1]; the ORDER and concurrency of the launches is what this shows. Usage: python tools/graph_timeline.py [cfg1]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
torch.cuda.set_device(0)
td3, shape, B = bench.build_td3(name, 1, 0, "auto", 200_000)
td3.update_pair(1)
w = _lib.Watch("*", 256)
w.arm()
td3.capture_pair()
n = w.used()
names = [pk.lib().spikerl_prof_watch_name(i).decode() for i in range(n)]
_lib.Watch.off()
for _ in range(5):
    td3.replay_pair()
torch.cuda.synchronize()
plain = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); td3.replay_pair(); e1.record(); torch.cuda.synchronize()
    plain.append(e0.elapsed_time(e1))
t0 = w.ev[0][0]
rows = []
for i in range(n):
    a, b = w.ev[i]
    rows.append((t0.elapsed_time(a) * 1e3, t0.elapsed_time(b) * 1e3, names[i]))
rows.sort()
end = max(r[1] for r in rows)
print(f"{name}: pair graph with {n} watched launches; this replay {end:.1f} us (median plain replay "
      f"{sorted(plain)[len(plain) // 2] * 1e3:.1f} us)")
for a, b, nm in rows:
    bar = " " * int(a / end * 60) + "#" * max(1, int((b - a) / end * 60))
    print(f"{a:8.1f} {b:8.1f} {b - a:7.1f}  {nm:24s} |{bar}")
