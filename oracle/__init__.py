"""SpikeRL hot-path ORACLE — plain, slow, obviously-correct CPU implementation (numpy).

*** TEST INFRASTRUCTURE ONLY. ***
Only tests/, __graft_entry__.smoke() and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import, call or execute anything under oracle/. The product path
(paper_2502_17496_b200/ + libspikerl.so) never imports it and has no CPU fallback.
The oracle shares no code with the CUDA path; inputs come from synthgen/ (seeded
generators only, no method arithmetic).

Modules (each cites the passages it follows):
  numerics.py  bf16 RNE emulation                       — pinned
  actor.py     encoder / LIF / decoder forward, BPTT backward — pinned
  critic.py    twin ReLU critic forward/backward (configs[1]) — pinned (FD)
  td3.py       TD3 update, Adam, Polyak          — pinned (arithmetic)
  dual.py      forward-mode dual-number second oracle for BPTT
  amp.py       dynamic loss scaling (GradScaler) state machine — pinned
Unpinned: learning dynamics / rewards (no environment; PAPER.md Figs 5a-c missing) — out of
scope, "parity unpinned".
"""
from .numerics import bf16, fp32, rounder  # noqa: F401
from .actor import (gaussian_stim, gaussian_stim_f64, encode_spikes, lif_layer_forward, decode, actor_forward,  # noqa: F401
                    surrogate, lif_reverse_scan, actor_backward, counts)
from .critic import critic_forward, critic_backward  # noqa: F401
from .td3 import adam_update, polyak, init_state, td3_update  # noqa: F401
from .amp import amp_step, unscale, all_finite  # noqa: F401
