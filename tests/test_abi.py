"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/spikerl.h declares, and the host-side validation / size / layout calls behave."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2502_17496_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib


def header_functions():
    src = open(os.path.join(ROOT, "include", "spikerl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spikerl_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_header_symbol(L):
    lib = L.lib()
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(L.EXPORTS)


def test_version_and_launch_counter(L):
    assert b"sm_100a" in L.lib().spikerl_version()
    L.lib().spikerl_launch_count(1)
    assert L.lib().spikerl_launch_count(0) == 0


def cfg(**kw):
    from paper_2502_17496_b200 import actor_cfg
    base = dict(obs_dim=17, act_dim=6, precision="fp32")
    base.update(kw)
    return actor_cfg(**base)


def test_param_offsets_layout(L):
    from paper_2502_17496_b200 import actor_offsets, critic_offsets, critic_cfg
    off = actor_offsets(cfg())
    S, E, N1, N2, A, D = 17, 10, 256, 256, 6, 10
    sizes = [S * E, S * E, N1 * S * E, N2 * N1, A * D * N2, A * D, A]
    assert off == [0] + list(__import__("itertools").accumulate(sizes))
    assert L.lib().spikerl_actor_param_count(C.byref(cfg())) == off[-1] == 124_822
    coff = critic_offsets(critic_cfg(23))
    assert coff[-1] == 23 * 256 + 256 + 256 * 256 + 256 + 256 + 1


@pytest.mark.parametrize("field,value,status", [
    ("T", 0, 2), ("T", 256, 2), ("d_c", 1.5, 2), ("d_v", -0.1, 2), ("v_th", 0.0, 2),
    ("surr_window", 0.0, 2), ("obs_dim", 0, 2), ("pop_enc", 0, 2), ("precision", 7, 1), ("engine", 9, 1)])
def test_cfg_validation(L, field, value, status):
    c = cfg()
    setattr(c, field, value)
    assert L.lib().spikerl_actor_cfg_check(C.byref(c)) == status
    assert len(L.last_error()) > 0
    assert L.lib().spikerl_actor_param_count(C.byref(c)) == 0


def test_reset_grad_validation_and_tape(L):
    """reset_grad (rho) is 0 or 1; rho = 1 adds the fp32 membrane planes [T][B][P_l] to the tape and
    is not offered for FP16 operands."""
    assert L.lib().spikerl_actor_cfg_check(C.byref(cfg(reset_grad=2))) == L.E_DOMAIN
    assert L.lib().spikerl_actor_cfg_check(C.byref(cfg(precision="fp16", reset_grad=1))) == L.E_UNSUPPORTED
    B = 64
    l0, l1 = L.TapeLayout(), L.TapeLayout()
    assert L.lib().spikerl_actor_tape_layout(C.byref(cfg(precision="bf16")), B, C.byref(l0)) == 0
    assert L.lib().spikerl_actor_tape_layout(C.byref(cfg(precision="bf16", reset_grad=1)), B, C.byref(l1)) == 0
    assert list(l0.V) == [0, 0, 0, 0] and all(l1.V[i] > 0 for i in (1, 2, 3))
    extra = sum(4 * 5 * B * l1.padded[i] for i in (1, 2, 3))
    assert l1.total - l0.total >= extra


def test_tcgen05_needs_bf16(L):
    c = cfg(engine="tcgen05")
    assert L.lib().spikerl_actor_cfg_check(C.byref(c)) == L.E_UNSUPPORTED


@pytest.mark.parametrize("T,status", [(5, 0), (16, 0), (24, 0), (17, 7), (33, 7)])
def test_auto_engine_never_switches_silently(L, T, status):
    """bf16 with ENGINE_AUTO runs on tcgen05; a shape it cannot tile is E_UNSUPPORTED (no silent drop
    to another engine: north_star "no multi-backend dispatch"); ENGINE_SIMT must then be asked for."""
    c = cfg(precision="bf16", T=T)
    assert L.lib().spikerl_actor_cfg_check(C.byref(c)) == status, L.last_error()
    assert L.lib().spikerl_actor_cfg_check(C.byref(cfg(precision="bf16", T=T, engine="simt"))) == 0


def test_bf16_critic_shape_not_silently_rerouted(L):
    """A bf16 critic outside the tensor-core kernels' shapes (hidden 256-256, in <= 512) is rejected on
    the host before anything is enqueued; fp32 critics run on the SIMT GEMMs; loss scaling needs bf16."""
    lib = L.lib()
    from paper_2502_17496_b200 import critic_cfg, td3_cfg
    for cc, st_expect in ((critic_cfg(23, hidden1=128, hidden2=128), L.E_UNSUPPORTED),
                          (critic_cfg(600), L.E_UNSUPPORTED)):
        z = C.c_void_p(256)
        st = lib.spikerl_critic_fwd_bwd(C.byref(cc), 8, z, z, z, cc.in_dim - 6, z, 6, None, z, None, None, None,
                                        0.0, z, None)
        assert st == st_expect, L.last_error()
    c = cfg(precision="fp32")
    cc = critic_cfg(23, precision="fp32")
    bufs = L.TD3Bufs()
    for f, _ in L.TD3Bufs._fields_:
        setattr(bufs, f, 256)
    bufs.fused_critic = bufs.fused_actor = None
    bufs.replay_size = 1000
    bufs.amp = 256
    st = lib.spikerl_td3_update(C.byref(c), C.byref(cc), C.byref(td3_cfg(256)), C.byref(bufs), 1, 0, None, None,
                                None, C.c_void_p(256), C.c_void_p(256), None)
    assert st == L.E_UNSUPPORTED, L.last_error()


def test_tape_layout_sizes(L):
    c = cfg(precision="bf16")
    lay = L.TapeLayout()
    B = 256
    assert L.lib().spikerl_actor_tape_layout(C.byref(c), B, C.byref(lay)) == 0
    assert list(lay.padded) == [256, 256, 256, 128]
    assert lay.total == L.lib().spikerl_actor_tape_bytes(C.byref(c), B)
    offs = [lay.A, *lay.bits, *lay.mask[1:], lay.counts, lay.act]
    assert all(o % 256 == 0 for o in offs) and sorted(offs) == offs
    assert lay.bits[1] - lay.bits[0] >= 5 * B * 8 * 4
    assert L.lib().spikerl_actor_tape_bytes(C.byref(c), 0) == 0


def test_sync_errors_enqueue_nothing(L):
    """Argument errors are reported on the host before any device work (no GPU needed)."""
    lib = L.lib()
    c = cfg()
    assert lib.spikerl_actor_forward(C.byref(c), 0, None, None, None, None, None, None, None) == L.E_ARG
    t = L.Tape(0, 0, 0, None, 0)
    assert lib.spikerl_actor_backward(C.byref(c), 4, C.c_void_p(16), None, C.c_void_p(16), C.byref(t),
                                      C.c_void_p(16), C.c_void_p(16), 0, C.c_void_p(16), None) == L.E_STATE
    assert lib.spikerl_adam(None, None, None, None, 0, None, 1e-3, 0.9, 0.999, 1e-8, 0, 0, 0.0, None) == L.E_ARG
    assert lib.spikerl_allreduce_grads(None, None, 10, None) == 0      # no comm: identity
    from paper_2502_17496_b200 import critic_cfg, td3_cfg
    cc = critic_cfg(23, precision="fp32")
    bufs = L.TD3Bufs()
    for f, _ in L.TD3Bufs._fields_:
        setattr(bufs, f, 256)
    bufs.amp = bufs.fused_critic = bufs.fused_actor = None
    bufs.replay_size = 10
    hp = td3_cfg(256)
    st = lib.spikerl_td3_update(C.byref(c), C.byref(cc), C.byref(hp), C.byref(bufs), 1, 0, None, None, None,
                                C.c_void_p(256), C.c_void_p(256), None)
    assert st == L.E_NOTREADY, L.last_error()


def test_workspace_sizes_host_only(L):
    """Workspace-size queries are host logic: they answer without a device (they also create the
    fork/join streams when one is present) and grow with the batch."""
    lib = L.lib()
    from paper_2502_17496_b200 import critic_cfg, td3_cfg
    c = cfg(precision="bf16")
    cc = critic_cfg(23)
    a1, a2 = lib.spikerl_actor_workspace_bytes(C.byref(c), 64), lib.spikerl_actor_workspace_bytes(C.byref(c), 256)
    assert 0 < a1 < a2
    w = lib.spikerl_td3_workspace_bytes(C.byref(c), C.byref(cc), 256)
    # the TD3 workspace holds the actor workspace, a tape and two critic workspaces (online + target)
    assert w > a2 + lib.spikerl_actor_tape_bytes(C.byref(c), 256) + 2 * lib.spikerl_critic_workspace_bytes(C.byref(cc), 256) - 1
    assert lib.spikerl_actor_workspace_bytes(C.byref(c), 0) == 0


@pytest.mark.parametrize("in_dim", [23, 119, 393, 512])
def test_critic_bf16_layout(L, in_dim):
    """spikerl_critic_bf16_layout (host only): the per-critic blocks W1p | W1T | W2T | W2 tile the bf16
    buffer spikerl_critic_bf16_bytes sizes, after the [2][P] plain copy; other critics are refused."""
    from paper_2502_17496_b200 import critic_cfg, critic_offsets
    c = critic_cfg(in_dim)
    o = (C.c_longlong * 8)()
    assert L.lib().spikerl_critic_bf16_layout(C.byref(c), o) == 0
    base, tb, w1p, w1t, w2t, w2, inp, inq = list(o)
    P = critic_offsets(c)[-1]
    H = 256
    assert base >= 2 * P and base % 8 == 0 and inp % 16 == 0 and inp >= in_dim and inq >= inp
    assert (w1p, w1t, w2t, w2) == (0, H * inp, H * inp + inq * H, H * inp + inq * H + H * H)
    assert tb == w2 + H * H
    assert L.lib().spikerl_critic_bf16_bytes(C.byref(c)) >= 2 * (base + 2 * tb)
    assert L.lib().spikerl_critic_bf16_layout(C.byref(critic_cfg(in_dim, precision="fp32")), o) != 0
