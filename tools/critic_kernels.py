"""Twin critic at one batch size, a few calls of each kind (forward, update fwd+bwd, actor step) for
an ncu launch list (diagnostics). Usage: python tools/critic_kernels.py [B] [S] [A]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen as sg
import paper_2502_17496_b200 as pk
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = int(sys.argv[2]) if len(sys.argv) > 2 else 376
A = int(sys.argv[3]) if len(sys.argv) > 3 else 17
cs = sg.CriticShape(S + A)
rng = np.random.default_rng(0)
c = pk.TwinCritic(pk.critic_cfg(S + A), B)
c.load(sg.critic_params(cs, rng), sg.critic_params(cs, rng))
obs = torch.randn(B, S, device="cuda"); act = torch.rand(B, A, device="cuda") * 2 - 1
y = torch.randn(B, device="cuda"); ga = torch.zeros(B, A, device="cuda")
for _ in range(3):
    c(obs, act)
    c(obs, act, y=y)
    c(obs, act, grad_act=ga, act_grad_scale=-1.0 / B)
torch.cuda.synchronize()
print("ok")
