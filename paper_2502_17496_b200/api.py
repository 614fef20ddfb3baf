"""Thin Python binding over libspikerl.so (include/spikerl.h).

Argument marshalling only: torch supplies device memory, streams and process groups; every step
of the hot path runs in the library's CUDA kernels. No CPU fallback: every call goes through
the C ABI and raises SpikeRLError on a non-OK status.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib

_PREC = {"fp32": L.FP32, "bf16": L.BF16, "fp16": L.FP16}
_ENG = {"auto": L.ENGINE_AUTO, "simt": L.ENGINE_SIMT, "tcgen05": L.ENGINE_TCGEN05}


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------------------------ configs
def actor_cfg(obs_dim, act_dim, pop_enc=10, pop_dec=10, hidden1=256, hidden2=256, T=5, d_c=0.5, d_v=0.75,
              v_th=0.5, surr_window=0.5, surr_height=1.0, sigma_floor=1e-3, precision="bf16",
              engine="auto", reset_grad=0) -> L.ActorCfg:
    return L.ActorCfg(obs_dim, act_dim, pop_enc, pop_dec, hidden1, hidden2, T, d_c, d_v, v_th, surr_window,
                      surr_height, sigma_floor, _PREC[precision], _ENG[engine], reset_grad)


def actor_cfg_from(shape, engine="auto", reset_grad=0) -> L.ActorCfg:
    """From any object with the problem-statement attributes (obs_dim, act_dim, pop_enc, ...)."""
    return actor_cfg(shape.obs_dim, shape.act_dim, shape.pop_enc, shape.pop_dec, shape.n1, shape.n2, shape.T,
                     shape.d_c, shape.d_v, shape.v_th, shape.surr_window, shape.surr_height, shape.sigma_floor,
                     shape.precision, engine, reset_grad)


def critic_cfg(in_dim, hidden1=256, hidden2=256, precision="bf16") -> L.CriticCfg:
    return L.CriticCfg(in_dim, hidden1, hidden2, _PREC[precision])


def td3_cfg(batch, gamma=0.99, tau=0.005, policy_noise=0.2, noise_clip=0.5, policy_delay=2, lr_actor=1e-4,
            lr_critic=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, amp_growth=2.0, amp_backoff=0.5,
            amp_interval=2000) -> L.TD3Cfg:
    return L.TD3Cfg(gamma, tau, policy_noise, noise_clip, policy_delay, lr_actor, lr_critic, beta1, beta2, eps,
                    batch, amp_growth, amp_backoff, amp_interval)


def actor_offsets(cfg):
    off = (C.c_size_t * (len(L.ACTOR_PARAMS) + 1))()
    check(lib().spikerl_actor_param_offsets(C.byref(cfg), off), "actor_param_offsets")
    return list(off)


def critic_offsets(cfg):
    off = (C.c_size_t * (len(L.CRITIC_PARAMS) + 1))()
    check(lib().spikerl_critic_param_offsets(C.byref(cfg), off), "critic_param_offsets")
    return list(off)


def _actor_shapes(cfg):
    S, A, E, D = cfg.obs_dim, cfg.act_dim, cfg.pop_enc, cfg.pop_dec
    K0, N3 = S * E, A * D
    return {"mu": (S, E), "sigma": (S, E), "W1": (cfg.hidden1, K0), "W2": (cfg.hidden2, cfg.hidden1),
            "W3": (N3, cfg.hidden2), "Wd": (A, D), "bd": (A,)}


def _critic_shapes(cfg):
    return {"W1": (cfg.hidden1, cfg.in_dim), "b1": (cfg.hidden1,), "W2": (cfg.hidden2, cfg.hidden1),
            "b2": (cfg.hidden2,), "W3": (1, cfg.hidden2), "b3": (1,)}


def pack(offsets, shapes, names, params: dict, device="cuda") -> torch.Tensor:
    flat = np.zeros(offsets[-1], np.float32)
    for i, k in enumerate(names):
        a = np.asarray(params[k], np.float32).reshape(-1)
        assert a.size == offsets[i + 1] - offsets[i], (k, a.size)
        flat[offsets[i]:offsets[i + 1]] = a
    return torch.from_numpy(flat).to(device)


def unpack(offsets, shapes, names, flat) -> dict:
    x = flat.detach().cpu().numpy() if isinstance(flat, torch.Tensor) else np.asarray(flat)
    return {k: x[offsets[i]:offsets[i + 1]].reshape(shapes[k]).copy() for i, k in enumerate(names)}


def pack_actor(cfg, params, device="cuda"):
    return pack(actor_offsets(cfg), _actor_shapes(cfg), L.ACTOR_PARAMS, params, device)


def unpack_actor(cfg, flat):
    return unpack(actor_offsets(cfg), _actor_shapes(cfg), L.ACTOR_PARAMS, flat)


def pack_critic(cfg, params, device="cuda"):
    return pack(critic_offsets(cfg), _critic_shapes(cfg), L.CRITIC_PARAMS, params, device)


def unpack_critic(cfg, flat):
    return unpack(critic_offsets(cfg), _critic_shapes(cfg), L.CRITIC_PARAMS, flat)


def unpack_bits(words: torch.Tensor, n: int) -> np.ndarray:
    """u32 bit plane [..., P/32] -> uint8 [..., n] (bit j of word w = neuron 32w + j)."""
    w = words.detach().cpu().numpy().astype(np.uint32)
    b = np.unpackbits(w.view(np.uint8).reshape(w.shape + (4,)), axis=-1, bitorder="little")
    return b.reshape(w.shape[:-1] + (w.shape[-1] * 32,))[..., :n]


def _alloc(nbytes, device="cuda"):
    return torch.zeros(max(int(nbytes), 16), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------------------------ actor
class SpikingActor:
    """Population-coded spiking actor driving the C-ABI forward/backward."""

    def __init__(self, cfg: L.ActorCfg, batch: int, device="cuda"):
        self.cfg, self.batch, self.device = cfg, batch, device
        check(lib().spikerl_actor_cfg_check(C.byref(cfg)), "actor cfg")
        self.offsets = actor_offsets(cfg)
        self.n_params = self.offsets[-1]
        self.params = torch.zeros(self.n_params, dtype=torch.float32, device=device)
        self.bf16 = cfg.precision in (L.BF16, L.FP16)
        self.params_bf16 = _alloc(lib().spikerl_actor_bf16_bytes(C.byref(cfg)), device) if self.bf16 else None
        self.tape_buf = _alloc(lib().spikerl_actor_tape_bytes(C.byref(cfg), batch), device)
        self.ws = _alloc(lib().spikerl_actor_workspace_bytes(C.byref(cfg), batch), device)
        self.tape = L.Tape(0, 0, 0, self.tape_buf.data_ptr(), self.tape_buf.numel())
        self.grads = torch.zeros(self.n_params, dtype=torch.float32, device=device)
        self.actions = torch.zeros(batch, cfg.act_dim, dtype=torch.float32, device=device)
        lay = L.TapeLayout()
        check(lib().spikerl_actor_tape_layout(C.byref(cfg), batch, C.byref(lay)), "tape layout")
        self.layout = lay

    def load(self, params: dict):
        self.params.copy_(pack_actor(self.cfg, params, self.device))
        self.refresh()

    def refresh(self):
        if self.bf16:
            check(lib().spikerl_actor_refresh_bf16(C.byref(self.cfg), _p(self.params), _p(self.params_bf16),
                                                   _stream()), "refresh_bf16")

    def forward(self, obs: torch.Tensor, record=True) -> torch.Tensor:
        assert obs.shape == (self.batch, self.cfg.obs_dim) and obs.dtype == torch.float32 and obs.is_contiguous()
        check(lib().spikerl_actor_forward(C.byref(self.cfg), self.batch, _p(self.params), _p(self.params_bf16),
                                          _p(obs), _p(self.actions), C.byref(self.tape) if record else None,
                                          _p(self.ws), _stream()), "actor_forward")
        return self.actions

    def backward(self, obs: torch.Tensor, grad_actions: torch.Tensor, accumulate=False, comm=None) -> torch.Tensor:
        """BPTT; with `comm` the gradient ends as the mean over ranks, allreduced per bucket while the
        backward still runs (spikerl_actor_backward_dp)."""
        if comm is None:
            check(lib().spikerl_actor_backward(C.byref(self.cfg), self.batch, _p(self.params), _p(self.params_bf16),
                                               _p(obs), C.byref(self.tape), _p(grad_actions), _p(self.grads),
                                               int(accumulate), _p(self.ws), _stream()), "actor_backward")
        else:
            check(lib().spikerl_actor_backward_dp(C.byref(self.cfg), self.batch, _p(self.params),
                                                  _p(self.params_bf16), _p(obs), C.byref(self.tape),
                                                  _p(grad_actions), _p(self.grads), int(accumulate), comm.handle,
                                                  _p(self.ws), _stream()), "actor_backward_dp")
        return self.grads

    def grad_buckets(self):
        """[0, off W2, off W3, total): the allreduce buckets of the flat gradient."""
        b = (C.c_size_t * 4)()
        check(lib().spikerl_actor_grad_buckets(C.byref(self.cfg), b), "grad_buckets")
        return list(b)

    # tape views (for parity tests / diagnostics)
    def tape_view(self):
        return tape_view(self.cfg, self.batch, self.tape_buf, 0)

    def inference_tape_view(self):
        """The tape an inference-only forward (forward(obs, record=False)) left in the workspace (its
        stimulation plane A is not written)."""
        off = lib().spikerl_actor_workspace_tape_offset(C.byref(self.cfg), self.batch)
        return tape_view(self.cfg, self.batch, self.ws, off)

    def spikes(self):
        """Host copies of the spike / mask planes as uint8 [T][B][N_l]."""
        return tape_spikes(self.cfg, self.tape_view())


def tape_view(cfg, B, buf, base=0):
    """Typed views of a tape held in the uint8 device buffer ``buf`` at byte offset ``base``
    (spikerl_actor_tape_layout), for parity tests / diagnostics."""
    lay = L.TapeLayout()
    check(lib().spikerl_actor_tape_layout(C.byref(cfg), B, C.byref(lay)), "tape layout")
    T = cfg.T
    K0, N3 = cfg.obs_dim * cfg.pop_enc, cfg.act_dim * cfg.pop_dec

    def seg(off, nbytes, dtype, shape):
        return buf[base + off:base + off + nbytes].view(dtype).view(*shape)
    out = {"A": seg(lay.A, 4 * B * K0, torch.float32, (B, K0))}
    for l in range(4):
        W = lay.padded[l] // 32
        out[f"bits{l}"] = seg(lay.bits[l], 4 * T * B * W, torch.int32, (T, B, W))
        if l:
            out[f"mask{l}"] = seg(lay.mask[l], 4 * T * B * W, torch.int32, (T, B, W))
        if l and lay.bitsT[l]:
            P = lay.padded[l]
            Q = (B + 31) // 32 * 8          # batch quads
            nb = Q * P * (lay.tpad // 2)
            out[f"bitsT{l}"] = seg(lay.bitsT[l], nb, torch.uint8, (Q, P, lay.tpad // 2))
            out[f"maskT{l}"] = seg(lay.maskT[l], nb, torch.uint8, (Q, P, lay.tpad // 2))
            # the tcgen05 engine keeps the hidden layers' window bits only quad-major (the
            # dX epilogue's input); this diagnostic view re-packs them batch-major
            out[f"mask{l}"] = _quads_to_words(out[f"maskT{l}"], T, B)
    for l in (1, 2, 3):
        if lay.V[l]:
            out[f"V{l}"] = seg(lay.V[l], 4 * T * B * lay.padded[l], torch.float32, (T, B, lay.padded[l]))
    out["counts"] = seg(lay.counts, B * N3, torch.uint8, (B, N3))
    out["act"] = seg(lay.act, 4 * B * cfg.act_dim, torch.float32, (B, cfg.act_dim))
    return out


def tape_spikes(cfg, v):
    """Host copies of a tape view's spike / mask planes as uint8 [T][B][N_l]."""
    N = [cfg.obs_dim * cfg.pop_enc, cfg.hidden1, cfg.hidden2, cfg.act_dim * cfg.pop_dec]
    o = {f"o{l}": unpack_bits(v[f"bits{l}"], N[l]) for l in range(4)}
    o.update({f"h{l}": unpack_bits(v[f"mask{l}"], N[l]) for l in (1, 2, 3)})
    return o


def _quads_to_words(qt, T, B):
    """Diagnostics only (tape views for tests): quad-major bytes [Q][P][Tpad/2] (nibble s of a
    (quad, neuron) row = its 4 batch rows at step s) -> batch-major int32 words [T][B][P/32]."""
    Q, P, half = qt.shape
    sh = torch.arange(8, device=qt.device, dtype=torch.uint8)
    bits = (qt.unsqueeze(-1) >> sh) & 1                               # [Q][P][Tpad/2][8]
    bits = bits.reshape(Q, P, 2 * half, 4).permute(2, 0, 3, 1)        # [Tpad][Q][4][P]
    bits = bits.reshape(2 * half, 4 * Q, P)[:T, :B].to(torch.int64)   # [T][B][P]
    w = (bits.reshape(T, B, P // 32, 32) << torch.arange(32, device=qt.device)).sum(-1)
    return torch.where(w >= 2 ** 31, w - 2 ** 32, w).to(torch.int32)


# ------------------------------------------------------------------------------------ critic
class TwinCritic:
    def __init__(self, cfg: L.CriticCfg, batch: int, device="cuda"):
        self.cfg, self.batch, self.device = cfg, batch, device
        self.offsets = critic_offsets(cfg)
        self.P = self.offsets[-1]
        self.params = torch.zeros(2 * self.P, dtype=torch.float32, device=device)
        self.bf16 = cfg.precision in (L.BF16, L.FP16)
        self.params_bf16 = _alloc(lib().spikerl_critic_bf16_bytes(C.byref(cfg)), device) if self.bf16 else None
        self.ws = _alloc(lib().spikerl_critic_workspace_bytes(C.byref(cfg), batch), device)
        self.q = torch.zeros(2, batch, dtype=torch.float32, device=device)
        self.loss = torch.zeros(1, dtype=torch.float32, device=device)
        self.grads = torch.zeros(2 * self.P, dtype=torch.float32, device=device)

    def load(self, p1: dict, p2: dict):
        self.params.copy_(torch.cat([pack_critic(self.cfg, p1, self.device), pack_critic(self.cfg, p2, self.device)]))
        self.refresh()

    def refresh(self):
        if self.bf16:
            check(lib().spikerl_critic_refresh_bf16(C.byref(self.cfg), 2, _p(self.params), _p(self.params_bf16),
                                                    _stream()), "critic refresh")

    def __call__(self, obs, act, y=None, want_param_grads=True, grad_act=None, act_grad_scale=1.0):
        check(lib().spikerl_critic_fwd_bwd(C.byref(self.cfg), self.batch, _p(self.params), _p(self.params_bf16),
                                           _p(obs), obs.shape[1], _p(act), act.shape[1], _p(y), _p(self.q),
                                           _p(self.loss), _p(self.grads) if (y is not None and want_param_grads)
                                           else None, _p(grad_act), act_grad_scale, _p(self.ws), _stream()),
              "critic_fwd_bwd")
        return self.q


# ------------------------------------------------------------------------------------ optimiser
def adam(params, grads, m, v, step_counter, lr, beta1=0.9, beta2=0.999, eps=1e-8, clamp=(0, 0, 0.0)):
    check(lib().spikerl_adam(_p(params), _p(grads), _p(m), _p(v), params.numel(), _p(step_counter), lr, beta1,
                             beta2, eps, clamp[0], clamp[1], clamp[2], _stream()), "adam")


def polyak(target, source, tau):
    check(lib().spikerl_polyak(_p(target), _p(source), target.numel(), tau, _stream()), "polyak")


# ------------------------------------------------------------------------------------ comm
class Comm:
    """NCCL communicator owned by libspikerl; torch.distributed supplies only the rendezvous."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist
        idbuf = (C.c_ubyte * 128)()
        if rank == 0:
            check(lib().spikerl_comm_get_unique_id(idbuf), "comm id")
        obj = [bytes(idbuf)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        idbuf = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib().spikerl_comm_init(rank, world, idbuf, C.byref(h)), "comm init")
        self.handle, self.rank, self.world = h, rank, world

    def allreduce_mean(self, grads: torch.Tensor):
        check(lib().spikerl_allreduce_grads(self.handle, _p(grads), grads.numel(), _stream()), "allreduce")

    def broadcast(self, params: torch.Tensor, root=0):
        check(lib().spikerl_broadcast_params(self.handle, _p(params), params.numel(), root, _stream()), "broadcast")

    def alloc(self, n: int) -> torch.Tensor:
        """n fp32 zeros in NCCL symmetric-capable memory (spikerl_comm_mem_alloc: ncclMemAlloc), for
        buffers a fused allreduce + Adam plan registers. Freed when the tensor's storage dies."""
        ptr = C.c_void_p()
        check(lib().spikerl_comm_mem_alloc(self.handle, 4 * n, C.byref(ptr)), "comm_mem_alloc")
        t = torch.as_tensor(_CommMem(self, ptr.value, n), device="cuda")
        t.zero_()
        return t

    def fused_adam(self, grads: torch.Tensor, params: torch.Tensor, use_multimem=True):
        """A fused gradient-mean + Adam plan over (grads, params), both from alloc()."""
        h = C.c_void_p()
        check(lib().spikerl_fused_adam_create(self.handle, _p(grads), _p(params), params.numel(), int(use_multimem),
                                              C.byref(h)), "fused_adam_create")
        return h

    def close(self):
        if self.handle:
            lib().spikerl_comm_destroy(self.handle)
            self.handle = None


class _CommMem:
    """__cuda_array_interface__ over an ncclMemAlloc'd buffer (kept alive by the tensor using it)."""

    def __init__(self, comm, ptr, n):
        self.comm, self.ptr = comm, ptr
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            if self.comm.handle:
                lib().spikerl_comm_mem_free(self.comm.handle, C.c_void_p(self.ptr))
        except Exception:
            pass


# ------------------------------------------------------------------------------------ TD3
@dataclass
class ReplayShard:
    s: torch.Tensor
    a: torch.Tensor
    r: torch.Tensor
    s2: torch.Tensor
    d: torch.Tensor

    @property
    def size(self):
        return self.r.numel()


class TD3:
    """Device-resident TD3 state + the C-ABI update."""

    def __init__(self, acfg: L.ActorCfg, ccfg: L.CriticCfg, hp: L.TD3Cfg, replay: ReplayShard, device="cuda",
                 seed=0, comm: Comm | None = None, loss_scale: float | None = None, fused: bool = False):
        """fused (needs comm): the gradient mean and Adam of both networks run as the one fused kernel over
        NCCL symmetric memory (spikerl_fused_allreduce_adam) instead of allreduce + Adam launches."""
        self.acfg, self.ccfg, self.hp, self.replay, self.device, self.seed, self.comm = \
            acfg, ccfg, hp, replay, device, seed, comm
        lb = lib()
        self.Pa = actor_offsets(acfg)[-1]
        self.Pc = critic_offsets(ccfg)[-1]
        f32 = dict(dtype=torch.float32, device=device)
        fused = bool(fused and comm is not None)
        sym = (lambda n: comm.alloc(n)) if fused else (lambda n: torch.zeros(n, **f32))
        self.actor, self.actor_t = sym(self.Pa), torch.zeros(self.Pa, **f32)
        self.critic, self.critic_t = sym(2 * self.Pc), torch.zeros(2 * self.Pc, **f32)
        self.m_actor, self.v_actor = torch.zeros(self.Pa, **f32), torch.zeros(self.Pa, **f32)
        self.m_critic, self.v_critic = torch.zeros(2 * self.Pc, **f32), torch.zeros(2 * self.Pc, **f32)
        self.grad_actor, self.grad_critic = sym(self.Pa), sym(2 * self.Pc)
        self.fused_plans = (comm.fused_adam(self.grad_critic, self.critic), comm.fused_adam(self.grad_actor, self.actor)) \
            if fused else (None, None)
        self.bf16 = acfg.precision in (L.BF16, L.FP16)
        ab = lb.spikerl_actor_bf16_bytes(C.byref(acfg))
        cb = lb.spikerl_critic_bf16_bytes(C.byref(ccfg))
        self.actor_bf16 = _alloc(ab, device) if self.bf16 else None
        self.actor_t_bf16 = _alloc(ab, device) if self.bf16 else None
        self.critic_bf16 = _alloc(cb, device) if self.bf16 else None
        self.critic_t_bf16 = _alloc(cb, device) if self.bf16 else None
        self.adam_steps = torch.zeros(4, dtype=torch.int64, device=device)
        self.rng_counter = torch.zeros(1, dtype=torch.int64, device=device)
        self.losses = torch.zeros(2, **f32)
        # dynamic loss scaling state (None: no scaling): {scale, finite steps, found_inf, -} x {critic, actor}
        self.amp = None
        if loss_scale is not None:
            self.amp = torch.zeros(8, **f32)
            self.amp[0] = loss_scale
            self.amp[4] = loss_scale
        self.ws = _alloc(lb.spikerl_td3_workspace_bytes(C.byref(acfg), C.byref(ccfg), hp.batch), device)
        self._bufs = L.TD3Bufs(*[t.data_ptr() if t is not None else None for t in (
            self.actor, self.actor_t, self.actor_bf16, self.actor_t_bf16, self.critic, self.critic_t,
            self.critic_bf16, self.critic_t_bf16, self.m_actor, self.v_actor, self.m_critic, self.v_critic,
            self.grad_actor, self.grad_critic, self.adam_steps, self.rng_counter, replay.s, replay.a, replay.r,
            replay.s2, replay.d)], replay.size, self.amp.data_ptr() if self.amp is not None else None,
            self.fused_plans[0], self.fused_plans[1])
        self.graphs = {}
        self.ws_pair = None
        self.pair_graph = None

    def load(self, actor: dict, critic1: dict, critic2: dict):
        a = pack_actor(self.acfg, actor, self.device)
        c = torch.cat([pack_critic(self.ccfg, critic1, self.device), pack_critic(self.ccfg, critic2, self.device)])
        self.actor.copy_(a); self.actor_t.copy_(a); self.critic.copy_(c); self.critic_t.copy_(c)
        if self.comm is not None:
            for t in (self.actor, self.actor_t, self.critic, self.critic_t):
                self.comm.broadcast(t, 0)          # PAPER.md:135 broadcast_weights
        self.refresh()

    def refresh(self):
        if not self.bf16:
            return
        lb, s = lib(), _stream()
        check(lb.spikerl_actor_refresh_bf16(C.byref(self.acfg), _p(self.actor), _p(self.actor_bf16), s), "r")
        check(lb.spikerl_actor_refresh_bf16(C.byref(self.acfg), _p(self.actor_t), _p(self.actor_t_bf16), s), "r")
        check(lb.spikerl_critic_refresh_bf16(C.byref(self.ccfg), 2, _p(self.critic), _p(self.critic_bf16), s), "r")
        check(lb.spikerl_critic_refresh_bf16(C.byref(self.ccfg), 2, _p(self.critic_t), _p(self.critic_t_bf16), s),
              "r")

    def bf16_maintained(self, target: bool) -> torch.Tensor:
        """Bool mask over the critic twin bf16 buffer (as int16 elements) of what the updates keep current:
        everything but the transposed blocks nothing reads (spikerl_critic_bf16_layout)."""
        n = self.critic_bf16.numel() // 2
        mask = torch.ones(n, dtype=torch.bool, device=self.critic_bf16.device)
        o = (C.c_longlong * 8)()
        if lib().spikerl_critic_bf16_layout(C.byref(self.ccfg), o) != 0:
            return mask
        base, tb, _, w1t, w2t, _, _, inq = list(o)
        H = 256
        S, A = self.acfg.obs_dim, self.acfg.act_dim
        for z in range(2):
            blk = base + z * tb
            rows = mask[blk + w1t: blk + w1t + inq * H].view(inq, H)
            rows[:] = False
            if not target:
                rows[S:S + A] = True
                continue
            mask[blk + w2t: blk + w2t + H * H] = False
        return mask

    def update(self, step: int, indices: torch.Tensor | None = None, noise: torch.Tensor | None = None):
        check(lib().spikerl_td3_update(C.byref(self.acfg), C.byref(self.ccfg), C.byref(self.hp), C.byref(self._bufs),
                                       step, self.seed, _p(indices), _p(noise),
                                       self.comm.handle if self.comm is not None else None, _p(self.losses),
                                       _p(self.ws), _stream()), "td3_update")

    def update_pair(self, step: int, indices: torch.Tensor | None = None, noise: torch.Tensor | None = None):
        """Updates step (odd) and step + 1 as one overlapped DAG (policy_delay 2); bitwise the same
        as update(step); update(step + 1). indices [2][B], noise [2][B][A] or None."""
        if self.ws_pair is None:
            self.ws_pair = _alloc(lib().spikerl_td3_pair_workspace_bytes(C.byref(self.acfg), C.byref(self.ccfg),
                                                                          self.hp.batch), self.device)
        check(lib().spikerl_td3_update_pair(C.byref(self.acfg), C.byref(self.ccfg), C.byref(self.hp),
                                            C.byref(self._bufs), step, self.seed, _p(indices), _p(noise),
                                            self.comm.handle if self.comm is not None else None, _p(self.losses),
                                            _p(self.ws_pair), _stream()), "td3_update_pair")

    def capture_pair(self):
        """Capture the overlapped two-update DAG (steps 2j + 1, 2j + 2) as one CUDA graph."""
        if self.ws_pair is None:
            self.ws_pair = _alloc(lib().spikerl_td3_pair_workspace_bytes(C.byref(self.acfg), C.byref(self.ccfg),
                                                                          self.hp.batch), self.device)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.update_pair(1)
            self.pair_graph = g
        torch.cuda.current_stream().wait_stream(s)

    def replay_pair(self):
        self.pair_graph.replay()

    def capture(self):
        """Capture one CUDA graph per phase of the policy delay (critic-only / critic+actor)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for k in range(1, self.hp.policy_delay + 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.update(k)
                self.graphs[k % self.hp.policy_delay] = g
        torch.cuda.current_stream().wait_stream(s)

    def replay_graph(self, step: int):
        self.graphs[step % self.hp.policy_delay].replay()

    def ws_view(self, pair=False, slot=0):
        """Typed views of the intermediates the last update left in its workspace
        (spikerl_td3_workspace_layout); pair=True: the pair workspace, slot 0 / 1 = update k / k + 1."""
        lay = L.TD3WsLayout()
        B, S, A = self.hp.batch, self.acfg.obs_dim, self.acfg.act_dim
        check(lib().spikerl_td3_workspace_layout(C.byref(self.acfg), C.byref(self.ccfg), B, C.byref(lay)), "ws layout")
        buf = self.ws_pair if pair else self.ws
        base = slot * lay.total if pair else 0

        def f32(off, *shape):
            n = int(np.prod(shape))
            return buf[base + off:base + off + 4 * n].view(torch.float32).view(*shape)
        out = dict(s=f32(lay.s, B, S), a=f32(lay.a, B, A), r=f32(lay.r, B), s2=f32(lay.s2, B, S), d=f32(lay.d, B),
                   a2=f32(lay.a2, B, A), at=f32(lay.at, B, A), api=f32(lay.api, B, A), y=f32(lay.y, B),
                   ga=f32(lay.ga, B, A))
        out["tape_pi"] = tape_view(self.acfg, B, buf, base + lay.tape_pi)
        out["tape_target"] = tape_view(self.acfg, B, buf, base + lay.tape_target)
        return out


def replay_fill(n, obs_dim, act_dim, seed=0, rank=0, p_done=0.01, device="cuda") -> ReplayShard:
    f32 = dict(dtype=torch.float32, device=device)
    sh = ReplayShard(torch.empty(n, obs_dim, **f32), torch.empty(n, act_dim, **f32), torch.empty(n, **f32),
                     torch.empty(n, obs_dim, **f32), torch.empty(n, **f32))
    check(lib().spikerl_replay_fill(_p(sh.s), _p(sh.a), _p(sh.r), _p(sh.s2), _p(sh.d), n, obs_dim, act_dim, p_done,
                                    seed, rank, _stream()), "replay_fill")
    return sh


def replay_from_host(batch: dict, device="cuda") -> ReplayShard:
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device)
    return ReplayShard(t(batch["s"]), t(batch["a"]), t(batch["r"]), t(batch["s2"]), t(batch["d"]))
