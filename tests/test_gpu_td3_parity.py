"""TD3 update parity: the CUDA path (spikerl_td3_update through the C ABI) against the oracle with the
teacher-forced protocol of SURVEY.md §8(c) C-4 step 7 (readings R22-R24,
R30). Every update k starts the oracle from the GPU's own state before k (parameters, Adam m and v,
step counts, targets), and every stage is fed the GPU's inputs to that stage:

  target path   pi'(s') forward teacher forced on the GPU's target tape (spikes, masks, actions);
                a~ = clip(a2 + clip(eps), +-1) from the GPU's a2; y = r + gamma (1 - d) min Q'(s', a~)
                from the GPU's a~
  critic step   loss and gradients of both critics at the GPU's y
  Adam          oracle Adam applied to the GPU's own gradient
  actor step    pi(s) forward teacher forced on the GPU's tape; dQ1/da from the GPU's post-critic
                parameters and pi(s); actor gradient by the oracle BPTT on the GPU tape with the
                GPU's dQ1/da; Adam + sigma floor; Polyak of both targets

Tolerances (no looser than north_star): gradients, y, losses and dQ1/da relative L2 <= 1e-2 (bf16) /
1e-4 (fp32); actions 2e-2 abs (bf16) / 1e-4 rel (fp32); spikes teacher forced (disagreement only
within 1e-5 of V_th); optimizer outputs at the fp32-arithmetic bound of R30 (a few ulp), which is
tighter than any north_star figure. Parameters of a network that must not move are compared bitwise.
"""
import numpy as np
import pytest

import oracle
import synthgen as sg
from tests._parity import check_actor, rel_l2

pytestmark = pytest.mark.gpu

ULP32 = 2.0 ** -23


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _f64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _state(td3):
    import torch
    torch.cuda.synchronize()
    names = ("actor", "actor_t", "critic", "critic_t", "m_actor", "v_actor", "m_critic", "v_critic", "grad_actor",
             "grad_critic")
    st = {n: getattr(td3, n).detach().cpu().numpy().copy() for n in names}
    st["steps"] = td3.adam_steps.cpu().numpy().copy()
    st["losses"] = td3.losses.cpu().numpy().astype(np.float64)
    return st


def _critics(pk, td3, flat):
    P = td3.Pc
    return [{k: v.astype(np.float64) for k, v in pk.unpack_critic(td3.ccfg, flat[i * P:(i + 1) * P]).items()}
            for i in range(2)]


def _actor(pk, td3, flat):
    return {k: v.astype(np.float64) for k, v in pk.unpack_actor(td3.acfg, flat).items()}


def _f32(x):
    """A hyper-parameter as the fp32 value the C ABI passes the kernels (spikerl_td3_cfg is fp32)."""
    return float(np.float32(x))


def check_adam(p_pre, g, m_pre, v_pre, t, lr, p, m, v, clamp=None, what=""):
    """Oracle Adam (fp64) on the GPU's fp32 gradient and pre-state vs the GPU's fp32 result (R30):
    m, v within 4 ulp of the magnitude of their two terms, p within 2 ulp of |p| plus 1e-5 of the
    step lr (the step's own fp32 rounding: a quotient, a square root, a bias correction)."""
    f = lambda x: np.asarray(x, np.float64)
    hp = sg.TD3Hyper()
    pr, mr, vr = oracle.adam_update(f(p_pre), f(g), f(m_pre), f(v_pre), t, _f32(lr), _f32(hp.beta1), _f32(hp.beta2),
                                    _f32(hp.eps))
    if clamp is not None:
        lo, hi, cmin = clamp
        pr[lo:hi] = np.maximum(pr[lo:hi], cmin)
    gm = np.abs(f(g))
    em = 4 * ULP32 * (0.9 * np.abs(f(m_pre)) + 0.1 * gm) + 1e-38
    ev = 4 * ULP32 * (0.999 * f(v_pre) + 0.001 * gm * gm) + 1e-38
    ep = 2 * ULP32 * np.abs(pr) + 1e-5 * lr
    for name, x, ref, e in (("m", m, mr, em), ("v", v, vr, ev), ("p", p, pr, ep)):
        d = np.abs(f(x) - ref)
        assert np.all(d <= e), (what, name, float((d / e).max()), int(np.argmax(d / e)))


def check_polyak(tgt_pre, src, tau, tgt, what=""):
    """theta' <- tau theta + (1 - tau) theta' (fp32: two products and a sum) within 3 ulp of its terms."""
    f = lambda x: np.asarray(x, np.float64)
    tau = _f32(tau)
    ref = oracle.polyak(f(tgt_pre), f(src), tau)
    e = 3 * ULP32 * (tau * np.abs(f(src)) + (1 - tau) * np.abs(f(tgt_pre))) + 1e-38
    d = np.abs(f(tgt) - ref)
    assert np.all(d <= e), (what, float((d / e).max()))


def _gpu_actor_view(pk, td3, tape, a):
    return dict(a=_f64(a), grads=None, sp=pk.tape_spikes(td3.acfg, tape), A=tape["A"].cpu().numpy(),
                counts=tape["counts"].cpu().numpy())


def run_td3_teacher_forced(preset, prec, B=None, nsteps=2, seed=7):
    import torch
    import paper_2502_17496_b200 as pk
    shape, cs_, B0 = sg.preset(preset)
    B = B or B0
    shape = sg.with_(shape, precision=prec)
    S, A = shape.obs_dim, shape.act_dim
    cs = sg.CriticShape(S + A, precision=prec)
    hp = sg.TD3Hyper()
    rng = np.random.default_rng(seed)
    actor = sg.actor_params(shape, rng)
    c1, c2 = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
    N = max(4 * B, 2048)
    rb = sg.replay_batch(rng, N, S, A)
    td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(S + A, precision=prec), pk.td3_cfg(B),
                 pk.replay_from_host(rb), seed=1)
    td3.load(actor, c1, c2)
    tol = 1e-4 if prec == "fp32" else 1e-2
    stats = []
    for k in range(1, nsteps + 1):
        pre = _state(td3)
        idx = rng.integers(0, N, B)
        eps = sg.target_noise(rng, B, A)
        td3.update(k, torch.from_numpy(idx).cuda(), torch.from_numpy(eps).cuda())
        post = _state(td3)
        ws = td3.ws_view()
        batch = {key: rb[key][idx] for key in rb}
        # a1: the gathered minibatch is the indexed replay rows, bit for bit
        for key in ("s", "a", "r", "s2", "d"):
            assert np.array_equal(ws[key].cpu().numpy(), batch[key]), key
        s, a, r, s2, d = (batch[x].astype(np.float64) for x in ("s", "a", "r", "s2", "d"))
        st = {"k": k}
        # ---- target path (a2): pi'(s') teacher forced on the GPU's target tape
        at_pre = _actor(pk, td3, pre["actor_t"])
        st["target"] = check_actor(_gpu_actor_view(pk, td3, ws["tape_target"], ws["a2"]), shape,
                                   {kk: v.astype(np.float32) for kk, v in at_pre.items()}, batch["s2"], None,
                                   a_stored=False)   # the target forward is spikes-only
        a2 = _f64(ws["a2"])
        at_ref = np.clip(a2 + np.clip(eps.astype(np.float64), -hp.noise_clip, hp.noise_clip), -1.0, 1.0)
        at = _f64(ws["at"])
        assert np.all(np.abs(at - at_ref) <= 2 * ULP32 * (np.abs(a2) + 0.5)), "target-policy smoothing"
        # ---- y from the GPU's a~ and the pre-step target critics
        ct_pre = _critics(pk, td3, pre["critic_t"])
        x2 = np.concatenate([s2, at], axis=1)
        q1t, _ = oracle.critic_forward(ct_pre[0], x2, prec)
        q2t, _ = oracle.critic_forward(ct_pre[1], x2, prec)
        y_ref = r + hp.gamma * (1.0 - d) * np.minimum(q1t, q2t)
        y = _f64(ws["y"])
        st["y_rel"] = rel_l2(y, y_ref)
        assert st["y_rel"] <= tol, st
        # ---- critic step at the GPU's y: loss, gradients, Adam
        c_pre = _critics(pk, td3, pre["critic"])
        x = np.concatenate([s, a], axis=1)
        loss_ref, grads_ref = 0.0, []
        for i in range(2):
            qi, cache = oracle.critic_forward(c_pre[i], x, prec)
            loss_ref += np.mean((qi - y) ** 2)
            g, _ = oracle.critic_backward(c_pre[i], cache, 2.0 * (qi - y) / B, prec)
            grads_ref.append(g)
        assert abs(post["losses"][0] - loss_ref) <= tol * abs(loss_ref), (k, post["losses"][0], loss_ref)
        g_gpu = _critics(pk, td3, post["grad_critic"])
        st["critic_grad_rel"] = {}
        for i in range(2):
            for key, gr in grads_ref[i].items():
                e = rel_l2(g_gpu[i][key].reshape(gr.shape), gr)
                st["critic_grad_rel"][f"{i}.{key}"] = e
                assert e <= tol, (k, i, key, e)
        t_c = int(pre["steps"][0]) + 1
        assert int(post["steps"][0]) == t_c
        check_adam(pre["critic"], post["grad_critic"], pre["m_critic"], pre["v_critic"], t_c, hp.lr_critic,
                   post["critic"], post["m_critic"], post["v_critic"], what=f"critic Adam k={k}")
        if k % hp.policy_delay == 0:
            # ---- actor step: pi(s) teacher forced, dQ1/da from the post-critic-step parameters
            p_pre = _actor(pk, td3, pre["actor"])
            api = _f64(ws["api"])
            c_post = _critics(pk, td3, post["critic"])
            qp, cache = oracle.critic_forward(c_post[0], np.concatenate([s, api], axis=1), prec)
            _, dx = oracle.critic_backward(c_post[0], cache, np.full(B, -1.0 / B), prec, need_param_grads=False)
            ga_ref = dx[:, S:]
            ga = _f64(ws["ga"])
            st["ga_rel"] = rel_l2(ga, ga_ref)
            assert st["ga_rel"] <= tol, st
            la_ref = -np.mean(qp)
            assert abs(post["losses"][1] - la_ref) <= tol * abs(la_ref) + 1e-7, (post["losses"][1], la_ref)
            gview = _gpu_actor_view(pk, td3, ws["tape_pi"], ws["api"])
            gview["grads"] = _actor(pk, td3, post["grad_actor"])
            st["actor"] = check_actor(gview, shape, {kk: v.astype(np.float32) for kk, v in p_pre.items()},
                                      batch["s"], ga)
            off = pk.actor_offsets(td3.acfg)
            t_a = int(pre["steps"][2]) + 1
            assert int(post["steps"][2]) == t_a
            check_adam(pre["actor"], post["grad_actor"], pre["m_actor"], pre["v_actor"], t_a, hp.lr_actor,
                       post["actor"], post["m_actor"], post["v_actor"],
                       clamp=(off[1], off[2], np.float32(shape.sigma_floor)), what=f"actor Adam k={k}")
            check_polyak(pre["actor_t"], post["actor"], hp.tau, post["actor_t"], "actor target")
            check_polyak(pre["critic_t"], post["critic"], hp.tau, post["critic_t"], "critic targets")
        else:
            for n in ("actor", "actor_t", "critic_t", "m_actor", "v_actor"):
                assert np.array_equal(pre[n], post[n]), (k, n)
            assert int(post["steps"][2]) == int(pre["steps"][2])
        stats.append(st)
    return stats


@pytest.mark.parametrize("preset,prec,B,nsteps", [
    ("cfg1", "fp32", 256, 4), ("cfg1", "bf16", 256, 4), ("cfg2", "bf16", 512, 2), ("cfg3s", "bf16", 100, 2),
    ("cfg3L", "bf16", 4096, 2), ("cfg1", "bf16", 37, 2)])
def test_td3_teacher_forced(preset, prec, B, nsteps):
    """Configs[1] (both precisions, four updates: Adam bias corrections at t = 1, 2), configs[2],
    configs[3] at both per-rank batches (B = 4096 runs the BT = 32 forward tiles and the tcgen05 critic
    weight gradients), and a ragged batch."""
    for st in run_td3_teacher_forced(preset, prec, B, nsteps):
        print(preset, prec, B, {k: v for k, v in st.items() if k not in ("target", "actor")})
