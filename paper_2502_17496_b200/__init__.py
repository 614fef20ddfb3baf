"""SpikeRL (arxiv 2502.17496) hot path on B200: spiking-actor TD3 update behind a C ABI.

libspikerl.so (csrc/, include/spikerl.h) holds every kernel; this package only marshals
arguments (api.py). Importing it does not touch the GPU; the first library call loads the .so
and fails loudly if it is missing (no CPU fallback).
"""
from ._lib import SpikeRLError, lib, EXPORTS  # noqa: F401
from .api import (actor_cfg, actor_cfg_from, critic_cfg, td3_cfg, actor_offsets, critic_offsets,  # noqa: F401
                  pack_actor, unpack_actor, pack_critic, unpack_critic, unpack_bits, SpikingActor, TwinCritic,
                  adam, polyak, Comm, TD3, ReplayShard, replay_fill, replay_from_host, tape_view, tape_spikes)

__all__ = ["SpikeRLError", "lib", "actor_cfg", "actor_cfg_from", "critic_cfg", "td3_cfg", "SpikingActor",
           "TwinCritic", "TD3", "Comm", "adam", "polyak", "replay_fill", "replay_from_host"]
