"""Phase timeline (CTA 0, %globaltimer ns) of the fused small-batch actor forward, warm launch."""
import os, sys, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk
from paper_2502_17496_b200 import _lib
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
shape, _, _ = sg.preset(name)
rng = np.random.default_rng(0)
a = pk.SpikingActor(pk.actor_cfg_from(shape), B)
a.load(sg.actor_params(shape, rng))
s = torch.from_numpy(sg.observations(rng, B, shape.obs_dim)).cuda()
for _ in range(3):
    a.forward(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    a.forward(s)
e1.record()
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
_lib.lib().spikerl_debug_fused_trace(buf)
v = list(buf)
names = ["entry", "after_init", "enc_done", "x0_issued", "x0_recv", "l1_start", "x1_issued", "x1_recv", "l2_start",
         "x2_issued", "x2_recv", "l3_start", "x3_issued", "x3_recv", "dec_start", "done"]
names = names[:13] + names[14:]   # stamp 13 = decoder start, 14 = done
print(json.dumps({"us_per_forward": e0.elapsed_time(e1) / 50 * 1000,
                  "phases_ns": {n: (x - v[0]) for n, x in zip(names, v) if x}}))
