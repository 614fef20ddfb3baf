"""ctypes view of include/spikerl.h (argument marshalling only).

The shared library is built in-tree (paper_2502_17496_b200/libspikerl.so). If it is missing the
import of this module raises: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPIKERL_LIB_PATH: diagnostics only (A/B timing of two builds of this library)
LIB_PATH = os.environ.get("SPIKERL_LIB_PATH") or os.path.join(_HERE, "libspikerl.so")

OK, E_ARG, E_DOMAIN, E_STATE, E_NOTREADY, E_CUDA, E_NCCL, E_UNSUPPORTED = range(8)
STATUS_NAMES = ["OK", "E_ARG", "E_DOMAIN", "E_STATE", "E_NOTREADY", "E_CUDA", "E_NCCL", "E_UNSUPPORTED"]
FP32, BF16, FP16 = 0, 1, 2
ENGINE_AUTO, ENGINE_SIMT, ENGINE_TCGEN05 = 0, 1, 2
ACTOR_PARAMS = ("mu", "sigma", "W1", "W2", "W3", "Wd", "bd")
CRITIC_PARAMS = ("W1", "b1", "W2", "b2", "W3", "b3")


class SpikeRLError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"spikerl {STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")


class ActorCfg(C.Structure):
    _fields_ = [("obs_dim", C.c_int), ("act_dim", C.c_int), ("pop_enc", C.c_int), ("pop_dec", C.c_int),
                ("hidden1", C.c_int), ("hidden2", C.c_int), ("T", C.c_int),
                ("d_c", C.c_float), ("d_v", C.c_float), ("v_th", C.c_float),
                ("surr_window", C.c_float), ("surr_height", C.c_float), ("sigma_floor", C.c_float),
                ("precision", C.c_int), ("engine", C.c_int), ("reset_grad", C.c_int)]


class CriticCfg(C.Structure):
    _fields_ = [("in_dim", C.c_int), ("hidden1", C.c_int), ("hidden2", C.c_int), ("precision", C.c_int)]


class TD3Cfg(C.Structure):
    _fields_ = [("gamma", C.c_float), ("tau", C.c_float), ("policy_noise", C.c_float),
                ("noise_clip", C.c_float), ("policy_delay", C.c_int), ("lr_actor", C.c_float),
                ("lr_critic", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("batch", C.c_int), ("amp_growth", C.c_float), ("amp_backoff", C.c_float),
                ("amp_interval", C.c_int)]


class TapeLayout(C.Structure):
    _fields_ = [("A", C.c_size_t), ("bits", C.c_size_t * 4), ("mask", C.c_size_t * 4),
                ("counts", C.c_size_t), ("act", C.c_size_t), ("total", C.c_size_t),
                ("padded", C.c_int * 4), ("bitsT", C.c_size_t * 4), ("maskT", C.c_size_t * 4),
                ("tpad", C.c_int), ("V", C.c_size_t * 4)]


class Tape(C.Structure):
    _fields_ = [("magic", C.c_ulonglong), ("cfg_hash", C.c_ulonglong), ("batch", C.c_int),
                ("dev", C.c_void_p), ("bytes", C.c_size_t)]


class TD3Bufs(C.Structure):
    _fields_ = [("actor", C.c_void_p), ("actor_t", C.c_void_p), ("actor_bf16", C.c_void_p),
                ("actor_t_bf16", C.c_void_p), ("critic", C.c_void_p), ("critic_t", C.c_void_p),
                ("critic_bf16", C.c_void_p), ("critic_t_bf16", C.c_void_p), ("m_actor", C.c_void_p),
                ("v_actor", C.c_void_p), ("m_critic", C.c_void_p), ("v_critic", C.c_void_p),
                ("grad_actor", C.c_void_p), ("grad_critic", C.c_void_p), ("adam_steps", C.c_void_p),
                ("rng_counter", C.c_void_p), ("rs", C.c_void_p), ("ra", C.c_void_p), ("rr", C.c_void_p),
                ("rs2", C.c_void_p), ("rd", C.c_void_p), ("replay_size", C.c_longlong), ("amp", C.c_void_p),
                ("fused_critic", C.c_void_p), ("fused_actor", C.c_void_p)]


class TD3WsLayout(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("s", "a", "r", "s2", "d", "a2", "at", "api", "y", "ga", "tape_pi",
                                         "tape_target", "total")]


class ProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("bound", C.c_int), ("launches", C.c_longlong),
                ("total_ms", C.c_double), ("flops", C.c_double), ("bytes", C.c_double)]


class ProfSpan(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("start_ms", C.c_double), ("end_ms", C.c_double)]


BOUND_NAMES = ("hbm", "tensor", "alu", "latency")


def prof_enable(on: bool):
    lib().spikerl_prof_enable(1 if on else 0)


class Watch:
    """Live timing of one named kernel inside a timed region (spikerl_prof_watch): up to n launches
    per arming, each bracketed by its own timing-event pair on the stream it is launched on."""

    def __init__(self, name: str, n: int):
        import torch
        self.name, self.n = name, n
        self.ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in self.ev:   # torch creates the CUDA event lazily, at its first record
            a.record()
            b.record()
        torch.cuda.synchronize()
        self.total_ms, self.launches = 0.0, 0

    def arm(self):
        b = (P * self.n)(*[C.c_void_p(e[0].cuda_event) for e in self.ev])
        e = (P * self.n)(*[C.c_void_p(x[1].cuda_event) for x in self.ev])
        check(lib().spikerl_prof_watch(self.name.encode(), b, e, self.n), "prof_watch")

    def used(self) -> int:
        return lib().spikerl_prof_watch_count()

    @staticmethod
    def off():
        lib().spikerl_prof_watch(None, None, None, 0)

    def collect(self, k: int):
        """Add the durations of the first k pairs (their launches have completed: call after a sync)."""
        for a, b in self.ev[:k]:
            self.total_ms += a.elapsed_time(b)
        self.launches += k


def prof_timeline():
    """Launches of the profiling pass in enqueue order: [(name, start_ms, end_ms)]."""
    n = lib().spikerl_prof_timeline(None, 0)
    if n < 0:
        raise SpikeRLError(E_CUDA, last_error())
    arr = (ProfSpan * max(n, 1))()
    lib().spikerl_prof_timeline(arr, n)
    return [(e.name.decode(), e.start_ms, e.end_ms) for e in arr[:n]]


def prof_summary():
    n = lib().spikerl_prof_summary(None, 0)
    if n < 0:
        raise SpikeRLError(E_CUDA, last_error())
    arr = (ProfEntry * max(n, 1))()
    lib().spikerl_prof_summary(arr, n)
    return [dict(name=e.name.decode(), bound=BOUND_NAMES[e.bound], launches=e.launches, total_ms=e.total_ms,
                 flops=e.flops, bytes=e.bytes) for e in arr[:n]]


P = C.c_void_p
SZ = C.c_size_t
I = C.c_int
F = C.c_float
LL = C.c_longlong
ULL = C.c_ulonglong
_SIGS = {
    "spikerl_actor_cfg_check": (I, [C.POINTER(ActorCfg)]),
    "spikerl_actor_param_offsets": (I, [C.POINTER(ActorCfg), C.POINTER(SZ)]),
    "spikerl_actor_param_count": (SZ, [C.POINTER(ActorCfg)]),
    "spikerl_critic_param_offsets": (I, [C.POINTER(CriticCfg), C.POINTER(SZ)]),
    "spikerl_critic_param_count": (SZ, [C.POINTER(CriticCfg)]),
    "spikerl_actor_bf16_bytes": (SZ, [C.POINTER(ActorCfg)]),
    "spikerl_critic_bf16_bytes": (SZ, [C.POINTER(CriticCfg)]),
    "spikerl_critic_bf16_layout": (C.c_int, [C.POINTER(CriticCfg), C.POINTER(C.c_longlong)]),
    "spikerl_actor_tape_bytes": (SZ, [C.POINTER(ActorCfg), I]),
    "spikerl_actor_workspace_bytes": (SZ, [C.POINTER(ActorCfg), I]),
    "spikerl_actor_workspace_tape_offset": (SZ, [C.POINTER(ActorCfg), I]),
    "spikerl_critic_workspace_bytes": (SZ, [C.POINTER(CriticCfg), I]),
    "spikerl_td3_workspace_bytes": (SZ, [C.POINTER(ActorCfg), C.POINTER(CriticCfg), I]),
    "spikerl_td3_pair_workspace_bytes": (SZ, [C.POINTER(ActorCfg), C.POINTER(CriticCfg), I]),
    "spikerl_actor_tape_layout": (I, [C.POINTER(ActorCfg), I, C.POINTER(TapeLayout)]),
    "spikerl_td3_workspace_layout": (I, [C.POINTER(ActorCfg), C.POINTER(CriticCfg), I, C.POINTER(TD3WsLayout)]),
    "spikerl_actor_refresh_bf16": (I, [C.POINTER(ActorCfg), P, P, P]),
    "spikerl_critic_refresh_bf16": (I, [C.POINTER(CriticCfg), I, P, P, P]),
    "spikerl_actor_forward": (I, [C.POINTER(ActorCfg), I, P, P, P, P, C.POINTER(Tape), P, P]),
    "spikerl_actor_backward": (I, [C.POINTER(ActorCfg), I, P, P, P, C.POINTER(Tape), P, P, I, P, P]),
    "spikerl_actor_backward_dp": (I, [C.POINTER(ActorCfg), I, P, P, P, C.POINTER(Tape), P, P, I, P, P, P]),
    "spikerl_actor_grad_buckets": (I, [C.POINTER(ActorCfg), C.POINTER(SZ)]),
    "spikerl_critic_fwd_bwd": (I, [C.POINTER(CriticCfg), I, P, P, P, I, P, I, P, P, P, P, P, F, P, P]),
    "spikerl_adam": (I, [P, P, P, P, SZ, P, F, F, F, F, SZ, SZ, F, P]),
    "spikerl_polyak": (I, [P, P, SZ, F, P]),
    "spikerl_lif_scan_forward": (I, [P, I, I, I, F, F, F, F, P, P, P]),
    "spikerl_td3_update": (I, [C.POINTER(ActorCfg), C.POINTER(CriticCfg), C.POINTER(TD3Cfg),
                               C.POINTER(TD3Bufs), LL, ULL, P, P, P, P, P, P]),
    "spikerl_td3_update_pair": (I, [C.POINTER(ActorCfg), C.POINTER(CriticCfg), C.POINTER(TD3Cfg),
                                    C.POINTER(TD3Bufs), LL, ULL, P, P, P, P, P, P]),
    "spikerl_replay_fill": (I, [P, P, P, P, P, LL, I, I, F, ULL, I, P]),
    "spikerl_comm_get_unique_id": (I, [P]),
    "spikerl_comm_init": (I, [I, I, P, C.POINTER(P)]),
    "spikerl_comm_destroy": (I, [P]),
    "spikerl_comm_world": (I, [P]),
    "spikerl_comm_rank": (I, [P]),
    "spikerl_allreduce_grads": (I, [P, P, SZ, P]),
    "spikerl_broadcast_params": (I, [P, P, SZ, I, P]),
    "spikerl_comm_mem_alloc": (I, [P, SZ, C.POINTER(P)]),
    "spikerl_comm_mem_free": (I, [P, P]),
    "spikerl_fused_adam_create": (I, [P, P, P, SZ, I, C.POINTER(P)]),
    "spikerl_fused_adam_destroy": (I, [P]),
    "spikerl_fused_allreduce_adam": (I, [P, P, P, P, F, F, F, F, SZ, SZ, F, P]),
    "spikerl_last_error": (C.c_char_p, []),
    "spikerl_version": (C.c_char_p, []),
    "spikerl_launch_count": (LL, [I]),
    "spikerl_prof_enable": (None, [I]),
    "spikerl_prof_summary": (I, [P, I]),
    "spikerl_prof_timeline": (I, [P, I]),
    "spikerl_prof_watch": (I, [C.c_char_p, C.POINTER(P), C.POINTER(P), I]),
    "spikerl_prof_watch_count": (I, []),
    "spikerl_prof_watch_name": (C.c_char_p, [I]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().spikerl_last_error().decode()


def check(status: int, what: str = ""):
    if status != OK:
        raise SpikeRLError(status, f"{what}: {last_error()}")
    return status
