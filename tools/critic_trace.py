"""Phase timeline (CTA (0,0), %globaltimer ns) of the critic data-backward launch in the actor step
of a configs[1] TD3 update (eager, warm)."""
import os, sys, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
shape, cs, B = sg.preset(name)
rng = np.random.default_rng(0)
replay = pk.replay_fill(100000, shape.obs_dim, shape.act_dim, seed=1)
td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(cs.in_dim), pk.td3_cfg(B), replay, seed=1)
td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
for k in range(1, 9):   # ends with an actor step: the last launch forms dQ1/da
    td3.update(k)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
_lib.lib().spikerl_debug_critic_trace(buf)
v = list(buf)
names = ["entry", "after_pdl", "d2s_ticket", "dZ2T", "l2_mma", "dZ1T", "grad_act"]
print(json.dumps({n: (x - v[0]) if x else None for n, x in zip(names, v)}))
