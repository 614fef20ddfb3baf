"""The README usage example, run as a smoke check (GPU)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg                      # seeded synthetic parameters / inputs (tests and bench)
import paper_2502_17496_b200 as pk

shape, _, B = sg.preset("cfg1")            # obs 17, act 6, pop 10/10, hidden 256-256, T=5, bf16
S, A = shape.obs_dim, shape.act_dim
rng = np.random.default_rng(0)
cs = sg.CriticShape(S + A)
td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(S + A), pk.td3_cfg(B),
             pk.replay_fill(1_000_000, S, A, seed=1), seed=2)   # device-resident replay shard
td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
td3.update(1); td3.update(2)               # spikerl_td3_update (policy delay 2)
td3.capture_pair()                         # updates 2j+1, 2j+2 as one CUDA graph
for _ in range(100):
    td3.replay_pair()
print(td3.losses.cpu())                    # critic MSE, actor loss of the last update

actor = pk.SpikingActor(pk.actor_cfg_from(shape), 256)   # the actor alone
actor.load(sg.actor_params(shape, rng))
obs = torch.randn(256, S, device="cuda")
a = actor.forward(obs)                     # records the spike tape
g = actor.backward(obs, torch.ones_like(a))   # flat fp32 gradient (BPTT, surrogate gradient)
