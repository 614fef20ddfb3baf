"""Phase timeline (%globaltimer ns, CTA 0) of the last fused critic-update launch of a TD3 update-pair
graph replay: entry, after the PDL wait, own F tile done, barrier 1, own W tasks done, barrier 2, Adam
done. Usage: python tools/fused_trace.py [cfg1] [reps]"""
import os, sys, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
shape, cs, B = sg.preset(name)
rng = np.random.default_rng(0)
replay = pk.replay_fill(100000, shape.obs_dim, shape.act_dim, seed=1)
td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(cs.in_dim), pk.td3_cfg(B), replay, seed=1)
td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
td3.update_pair(1)
td3.capture_pair()
names = ["entry", "after_pdl", "F", "bar1", "W", "bar2", "adam", "w_staged", "x_tile", "l1", "w2_staged", "q", "dq", "dH1", "w_mma", "w_bias"]
rows = []
for _ in range(reps):
    for _ in range(50):   # back to back: clocks under load, as in the bench loop
        td3.replay_pair()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    _lib.lib().spikerl_debug_critic_trace(buf)
    v = list(buf)
    rows.append([(x - v[0]) for x in v[:16]])
med = [sorted(r[i] for r in rows)[len(rows) // 2] for i in range(16)]
print(json.dumps({"workload": name, "G": os.environ.get("SPIKERL_CRITIC_FUSED_G", "default"),
                  "ns_since_entry": dict(zip(names, med))}))
