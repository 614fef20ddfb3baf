"""Time the two TD3 step graphs (critic-only step, critic+actor step) separately at configs[1]."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
shape, cs, B = sg.preset(name)
rng = np.random.default_rng(0)
replay = pk.replay_fill(200000, shape.obs_dim, shape.act_dim, seed=1)
td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(cs.in_dim), pk.td3_cfg(B), replay, seed=1)
td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
for k in range(1, 5):
    td3.update(k)
td3.capture()
out = {}
for k, label in ((1, "critic_only"), (2, "critic_and_actor")):
    for _ in range(20):
        td3.replay_graph(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        td3.replay_graph(k)
    e1.record()
    torch.cuda.synchronize()
    out[label] = round(e0.elapsed_time(e1) / 200 * 1000, 2)
td3.capture_pair()
for _ in range(20):
    td3.replay_pair()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    td3.replay_pair()
e1.record()
torch.cuda.synchronize()
out["pair_per_update"] = round(e0.elapsed_time(e1) / 200 * 1000, 2)
print(json.dumps({"workload": name, "us_per_step": out, "serial": os.environ.get("SPIKERL_TD3_SERIAL", "0")}))
