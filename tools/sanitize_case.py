"""A small run of every kernel family for compute-sanitizer (one tool per call: racecheck or
synccheck; see B200_PROFILING.md): the fp32 SIMT actor (configs[0] B = 100), the bf16 tcgen05
actor (configs[1] widths, B = 64) forward + BPTT, a TD3 update pair (configs[1], B = 64), the
tcgen05 critic forced at B = 512 (SPIKERL_CRITIC_TC=2 from the caller). Diagnostic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
for name, B in (("cfg0", 100), ("cfg1", 64)):
    shape, _, _ = sg.preset(name)
    a = pk.SpikingActor(pk.actor_cfg_from(shape), B)
    a.load(sg.actor_params(shape, rng))
    obs = torch.from_numpy(sg.observations(rng, B, shape.obs_dim)).cuda()
    ga = torch.from_numpy(sg.action_grads(rng, B, shape.act_dim)).cuda()
    a.forward(obs); a.backward(obs, ga)
shape, cs, _ = sg.preset("cfg1")
replay = pk.replay_fill(4096, 17, 6, seed=1)
td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(23), pk.td3_cfg(64), replay, seed=1)
td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
td3.update_pair(1)
c = pk.TwinCritic(pk.critic_cfg(393), 512)
c.load(sg.critic_params(sg.CriticShape(393), rng), sg.critic_params(sg.CriticShape(393), rng))
obs = torch.randn(512, 376, device="cuda"); act = torch.rand(512, 17, device="cuda")
ga = torch.zeros(512, 17, device="cuda")
c(obs, act, torch.randn(512, device="cuda"))
c(obs, act, None, grad_act=ga, act_grad_scale=-1.0 / 512)
torch.cuda.synchronize()
print("sanitize case ok")
