"""Pins for the oracle (-m "not gpu"): the oracle is checked against what the paper, SPEC.md
and mathematics fix — hand traces, closed forms, special cases, an independent forward-mode
dual-number oracle and finite differences — never against itself.
"""
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
from oracle import dual
import synthgen as sg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def cfg_ns(**kw):
    base = dict(T=5, d_c=0.5, d_v=0.75, v_th=0.5, surr_window=0.5, surr_height=1.0,
                precision="fp32", obs_dim=1, act_dim=1, sigma_floor=1e-3)
    base.update(kw)
    return SimpleNamespace(**base)


# ------------------------------------------------------------------ bf16 rounding
def test_bf16_rne_laws():
    assert oracle.bf16(1.0 + 2.0 ** -8) == 1.0                      # tie -> even
    assert oracle.bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6      # tie -> even (up)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(1_000_000) * np.exp(rng.uniform(-20, 20, 1_000_000))
    r = oracle.bf16(x)
    assert np.array_equal(oracle.bf16(r), r)                        # idempotent
    xs = np.sort(x)
    assert np.all(np.diff(oracle.bf16(xs)) >= 0)                    # monotone
    assert np.all(np.abs(r - x) <= 2.0 ** -8 * np.abs(x) * (1 + 1e-7))  # |x - rn(x)| <= 2^-8 |x|


# ------------------------------------------------------------------ encoder
def test_gaussian_closed_form():
    mu = np.array([[1.0]], np.float32)
    sgm = np.array([[0.5]], np.float32)
    assert oracle.gaussian_stim(np.array([[1.0]], np.float32), mu, sgm)[0, 0] == 1.0      # s = mu
    A = oracle.gaussian_stim(np.array([[1.5]], np.float32), mu, sgm)[0, 0]              # s - mu = sigma
    assert A == np.float32(np.exp(-0.5))
    assert abs(float(A) - 0.606531) < 1e-6


def test_gaussian_symmetry_and_peak():
    mu = np.array([[0.25]], np.float32); sgm = np.array([[0.7]], np.float32)
    d = np.linspace(0, 3, 101).astype(np.float32)
    up = oracle.gaussian_stim((0.25 + d)[:, None].astype(np.float32), mu, sgm)[:, 0]
    dn = oracle.gaussian_stim((0.25 - d)[:, None].astype(np.float32), mu, sgm)[:, 0]
    # symmetric where 0.25 +- d are exact in fp32 (dyadic grid)
    dd = (np.arange(0, 49) / 16).astype(np.float32)
    assert np.array_equal(oracle.gaussian_stim((0.25 + dd)[:, None], mu, sgm),
                          oracle.gaussian_stim((0.25 - dd)[:, None], mu, sgm))
    assert up.max() == 1.0 and up[0] == 1.0 and np.all(np.diff(up) <= 0) and np.all(np.diff(dn) <= 0)


def test_mu_grid_recipe():
    p = sg.actor_params(sg.ActorShape(1, 1), np.random.default_rng(0))
    mu = p["mu"][0]
    assert mu[0] == -3 and mu[3] == -1 and mu[6] == 1 and mu[9] == 3
    assert float(mu[1]) == -2.3333332538604736
    assert float(mu[4]) == -0.3333333432674408 and float(mu[5]) == 0.3333333432674408


def _pattern(bits):
    return "".join(str(int(b)) for b in bits)


def test_encoder_pins_1d():
    g = gold("encoder_1d.json")
    p = sg.actor_params(sg.ActorShape(1, 1), np.random.default_rng(0))
    for case in g["cases"]:
        s = np.array([[case["s"]]], np.float32)
        A = oracle.gaussian_stim(s, p["mu"], p["sigma"])
        O = oracle.encode_spikes(A, g["T"])
        for n in case["neuron"]:
            assert abs(float(A[0, n]) - case["A"]) < 5e-7, (case, A[0, n])
            assert _pattern(O[:, 0, n]) == case["pattern"], case
            # closed form o_t = floor(tA) - floor((t-1)A) away from fp boundaries
            t = np.arange(1, g["T"] + 1)
            cf = np.floor(t * float(A[0, n])) - np.floor((t - 1) * float(A[0, n]))
            assert _pattern(cf.astype(int)) == case["pattern"]
        # all other population neurons silent at T=5 except those listed
        others = [e for e in range(10) if e not in case["neuron"]]
        if case["pattern"] == "00000":
            assert O[:, 0, :].sum() == 0
        else:
            assert O[:, 0, others].sum() == 0
    for ex in g["spec_examples"]:
        O = oracle.encode_spikes(np.array([[ex["A"]]], np.float32), ex["T"])
        assert _pattern(O[:, 0, 0]) == ex["pattern"]


def test_encoder_closed_form_dyadic():
    # A on a 2^-12 grid: fp32 accumulation is exact, so the closed form holds exactly
    rng = np.random.default_rng(1)
    A = (rng.integers(0, 4097, size=(64, 37)) / 4096.0).astype(np.float32)
    for T in (1, 2, 5, 16, 31):
        O = oracle.encode_spikes(A, T).astype(np.int64)
        t = np.arange(1, T + 1)[:, None, None]
        cf = np.floor(t * A.astype(np.float64)) - np.floor((t - 1) * A.astype(np.float64))
        assert np.array_equal(O, cf.astype(np.int64))
        assert np.array_equal(O.sum(0), np.floor(T * A.astype(np.float64)).astype(np.int64))


def test_encoder_count_monotone():
    A = np.linspace(0, 1, 2001).astype(np.float32)[None, :]
    for T in (3, 5, 16):
        c = oracle.encode_spikes(A, T).sum(axis=0)[0]
        assert np.all(np.diff(c.astype(int)) >= 0) and c.max() == T


# ------------------------------------------------------------------ LIF (north_star)
def test_lif_single_neuron_trace():
    g = gold("lif_neuron.json")
    o_in = np.ones((g["T"], 1, 1), np.uint8)
    V, O, I = oracle.lif_layer_forward(o_in, np.array([[g["I"]]]), 0.5, 0.75, 0.5)
    assert np.array_equal(V[:, 0, 0], np.array(g["v"]))
    assert np.array_equal(O[:, 0, 0], np.array(g["o"]))
    c = np.zeros(g["T"]); cc = 0.0
    for t in range(g["T"]):
        cc = 0.5 * cc + g["I"]; c[t] = cc
    assert np.array_equal(c, np.array(g["c"]))
    two = g["spec_two_step"]
    V2, O2, _ = oracle.lif_layer_forward(np.array([[[1]], [[0]]], np.uint8), np.array([[0.6]]),
                                         0.5, 0.75, 0.5)
    assert np.allclose(V2[:, 0, 0], two["v"], rtol=0, atol=1e-15)
    assert list(O2[:, 0, 0]) == two["o"]


def test_lif_special_cases():
    rng = np.random.default_rng(3)
    W = rng.standard_normal((7, 9))
    # zero input forever -> silent
    V, O, _ = oracle.lif_layer_forward(np.zeros((6, 4, 9), np.uint8), W, 0.5, 0.75, 0.5)
    assert O.sum() == 0 and np.all(V == 0)
    # d_v = 0 -> v_t == c_t
    o_in = (rng.random((6, 4, 9)) < 0.3).astype(np.uint8)
    V, O, I = oracle.lif_layer_forward(o_in, W, 0.5, 0.0, 0.5)
    c = np.zeros((4, 7)); cs = []
    for t in range(6):
        c = 0.5 * c + o_in[t] @ W.T; cs.append(c)
    assert np.allclose(V, np.array(cs), rtol=0, atol=1e-13)


def test_lif_backward_single_neuron():
    g = gold("lif_neuron.json")
    V = np.array(g["v"])[:, None, None]; O = np.array(g["o"], np.uint8)[:, None, None]
    gout = np.ones_like(V)
    G = oracle.lif_reverse_scan(gout, V, O, 0.5, 0.75, 0.5, 0.5, 1.0, rho=0.0)
    assert np.array_equal(G[:, 0, 0], np.array(g["G_z1_rho0"]))
    assert G.sum() == 10.125
    Gh = oracle.lif_reverse_scan(gout, V, O, 0.5, 0.75, 0.5, 0.5, 0.5, rho=0.0)
    assert np.array_equal(Gh, 0.5 * G)
    G1 = oracle.lif_reverse_scan(gout, V, O, 0.5, 0.75, 0.5, 0.5, 1.0, rho=1.0)
    assert np.allclose(G1[:, 0, 0], g["G_z1_rho1"], rtol=1e-15, atol=0)


# ------------------------------------------------------------------ golden tiny network
def _tiny(T=4, **kw):
    g = gold("tiny_net.json")
    p = {k: np.array(v, np.float32) for k, v in g["params"].items()}
    p.update({k: np.array(v, np.float32) for k, v in kw.items()})
    cfg = cfg_ns(T=T)
    return g, p, cfg


def test_golden_tiny_forward():
    g, p, cfg = _tiny()
    a, tape = oracle.actor_forward(p, cfg, np.array(g["s"], np.float32))
    f = g["forward"]
    assert np.array_equal(tape["A"][0], np.array(f["A"], np.float32))
    assert np.array_equal(tape["O0"][:, 0, :], np.array(f["enc_spikes"]))
    for l, (vk, ok) in enumerate((("v1", "o1"), ("v2", "o2"), ("v3", "o3"))):
        assert np.array_equal(tape["V"][l][:, 0, :], np.array(f[vk])), vk
        assert np.array_equal(tape["O"][l][:, 0, :], np.array(f[ok])), ok
    assert np.array_equal(tape["fr"][0], np.array(f["fr"]))
    assert tape["pre"][0, 0] == f["pre"]
    assert a[0, 0] == f["a"] == np.tanh(0.375)


@pytest.mark.parametrize("rho", [0.0, 1.0])
def test_golden_tiny_backward(rho):
    g, p, cfg = _tiny()
    a, tape = oracle.actor_forward(p, cfg, np.array(g["s"], np.float32))
    gr = oracle.actor_backward(p, cfg, tape, np.array(g["g_a"]), rho=rho)
    ref = dict(g["grads_rho0"])
    if rho:
        ref.update(g["grads_rho1"])
    for k, v in ref.items():
        assert np.allclose(gr[k], np.array(v), rtol=0, atol=5e-12), (k, gr[k], v)
    # mu/sigma: exactly 0 for the neuron with s == mu; < 1e-11 for the other
    assert gr["mu"][0, 1] == 0 and gr["sigma"][0, 1] == 0
    assert abs(gr["mu"][0, 0]) < 1e-11 and abs(gr["sigma"][0, 0]) < 1e-11


def test_T1_closed_form_golden():
    g, p, cfg = _tiny(T=1, W1=gold("tiny_net.json")["T1_variant"]["W1"])
    t1 = g["T1_variant"]
    a, tape = oracle.actor_forward(p, cfg, np.array(g["s"], np.float32))
    for l, (vk, ok) in enumerate((("v1", "o1"), ("v2", "o2"), ("v3", "o3"))):
        assert np.array_equal(tape["V"][l][0, 0], np.array(t1[vk]))
        assert np.array_equal(tape["O"][l][0, 0], np.array(t1[ok]))
    assert a[0, 0] == t1["a"]
    gr = oracle.actor_backward(p, cfg, tape, np.array(g["g_a"]))
    assert abs(gr["bd"][0] - t1["bd"]) < 1e-11 and abs(gr["Wd"][0, 0] - t1["Wd00"]) < 1e-11
    assert np.allclose(gr["W3"], t1["W3"], atol=1e-11, rtol=0)
    for k in ("W2", "W1", "mu", "sigma"):
        assert np.all(gr[k] == 0), k


def test_T1_is_heaviside_mlp():
    rng = np.random.default_rng(5)
    shp = sg.ActorShape(3, 2, pop_enc=4, pop_dec=3, n1=8, n2=6, T=1)
    for _ in range(10):
        p = sg.randomize_actor(shp, rng, scale=2.0)
        s = rng.standard_normal((5, 3)).astype(np.float32)
        a, tape = oracle.actor_forward(p, shp, s)
        A = oracle.gaussian_stim(s, p["mu"], p["sigma"]).astype(np.float64)
        x = (A >= 1.0).astype(np.float64)          # fires at T=1 iff A == 1 (s == mu)
        for l, W in enumerate((p["W1"], p["W2"], p["W3"])):
            x = (x @ W.astype(np.float64).T > 0.5).astype(np.float64)
            assert np.array_equal(tape["O"][l][0], x.astype(np.uint8))
        fr = x.reshape(5, 2, 3)
        assert np.allclose(a, np.tanh((fr * p["Wd"][None]).sum(-1) + p["bd"]), atol=1e-15)


# ------------------------------------------------------------------ zero cases (north_star)
def test_zero_decoder_weights_give_bias():
    rng = np.random.default_rng(7)
    shp = sg.ActorShape(4, 3, pop_enc=5, pop_dec=4, n1=16, n2=12, T=5)
    p = sg.randomize_actor(shp, rng, scale=3.0)
    p["Wd"] = np.zeros_like(p["Wd"])
    s = sg.observations(rng, 9, 4)
    a, tape = oracle.actor_forward(p, shp, s)
    assert np.array_equal(a, np.tile(np.tanh(p["bd"].astype(np.float64)), (9, 1)))
    g_a = sg.action_grads(rng, 9, 3)
    gr = oracle.actor_backward(p, shp, tape, g_a)
    for k in ("mu", "sigma", "W1", "W2", "W3"):
        assert np.all(gr[k] == 0), k
    tb = np.tanh(p["bd"].astype(np.float64))
    assert np.allclose(gr["bd"], (g_a.astype(np.float64) * (1 - tb * tb)).sum(0), rtol=1e-14)
    gpre = g_a.astype(np.float64) * (1 - tb * tb)
    assert np.allclose(gr["Wd"], (gpre[:, :, None] * tape["fr"].reshape(9, 3, 4)).sum(0), rtol=1e-14)


def test_zero_network_and_zero_cotangent():
    rng = np.random.default_rng(8)
    shp = sg.ActorShape(4, 3, pop_enc=5, pop_dec=4, n1=16, n2=12, T=5)
    p = sg.randomize_actor(shp, rng)
    for k in ("W1", "W2", "W3", "Wd", "bd"):
        p[k] = np.zeros_like(p[k])
    s = sg.observations(rng, 6, 4)
    a, tape = oracle.actor_forward(p, shp, s)
    assert np.all(a == 0) and all(o.sum() == 0 for o in tape["O"])
    p = sg.randomize_actor(shp, rng, scale=3.0)
    a, tape = oracle.actor_forward(p, shp, s)
    gr = oracle.actor_backward(p, shp, tape, np.zeros((6, 3)))
    assert all(np.all(v == 0) for v in gr.values())


def test_decoder_spec_example():
    O3 = np.zeros((5, 1, 2), np.uint8); O3[:, 0, 0] = 1
    a, fr, _ = oracle.decode(O3, np.array([[1.0, 1.0]]), np.array([0.0]), 5)
    assert a[0, 0] == np.tanh(1.0) and abs(a[0, 0] - 0.761594) < 1e-6


# ------------------------------------------------------------------ BPTT vs forward-mode duals
@pytest.mark.parametrize("seed", range(25))
def test_bptt_matches_forward_mode_duals(seed):
    rng = np.random.default_rng(100 + seed)
    T = int(rng.integers(1, 6))
    z = [1.0, 0.5][seed % 2]
    rho = [0.0, 1.0][(seed // 2) % 2]
    shp = sg.ActorShape(int(rng.integers(1, 4)), 2, pop_enc=4, pop_dec=4, n1=8, n2=6, T=T,
                        surr_height=z)
    p = sg.randomize_actor(shp, rng, scale=2.5)
    s = rng.uniform(-1, 1, size=(3, shp.obs_dim)).astype(np.float32)
    g_a = rng.standard_normal((3, 2))
    a, tape = oracle.actor_forward(p, shp, s)
    gr = oracle.actor_backward(p, shp, tape, g_a, rho=rho)
    gd, a_d = dual.actor_grads_forward_mode(p, shp, s, g_a, rho=rho)
    assert np.allclose(a, a_d, rtol=0, atol=1e-14)
    for k in gr:
        ref = gd[k]
        err = np.abs(gr[k] - ref).max()
        assert err <= 1e-6 * max(1.0, np.abs(ref).max()), (k, err)


def test_surrogate_height_homogeneity():
    # detached reset: dWd, dbd ~ z^0; dW3 ~ z; dW2 ~ z^2; dW1, dmu, dsigma ~ z^3 (R10)
    rng = np.random.default_rng(11)
    shp = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5)
    p = sg.randomize_actor(shp, rng, scale=2.5)
    s = rng.uniform(-1, 1, size=(4, 3)).astype(np.float32)
    g_a = rng.standard_normal((4, 2))
    a, tape = oracle.actor_forward(p, shp, s)
    g1 = oracle.actor_backward(p, shp, tape, g_a)
    g2 = oracle.actor_backward(p, sg.with_(shp, surr_height=0.5), tape, g_a)
    powers = dict(Wd=0, bd=0, W3=1, W2=2, W1=3, mu=3, sigma=3)
    for k, pw in powers.items():
        assert np.allclose(g2[k], g1[k] * 0.5 ** pw, rtol=1e-12, atol=1e-300), k


# ------------------------------------------------------------------ finite differences
@pytest.mark.parametrize("seed", range(10))
def test_critic_finite_differences(seed):
    rng = np.random.default_rng(200 + seed)
    cs = sg.CriticShape(7, 9, 8, precision="fp32")
    p = {k: v.astype(np.float64) for k, v in sg.critic_params(cs, rng).items()}
    for k in ("b1", "b2", "b3"):
        p[k] = rng.uniform(-0.3, 0.3, size=p[k].shape)
    x = rng.standard_normal((5, 7))
    w = rng.standard_normal(5)
    Q, cache = oracle.critic_forward(p, x)
    g, dx = oracle.critic_backward(p, cache, w)
    h = 1e-5
    L = lambda pp, xx: float((oracle.critic_forward(pp, xx)[0] * w).sum())
    for k in p:
        fd = np.zeros_like(p[k])
        for idx in np.ndindex(p[k].shape):
            pp = {kk: vv.copy() for kk, vv in p.items()}
            pp[k][idx] += h; lp = L(pp, x)
            pp[k][idx] -= 2 * h; lm = L(pp, x)
            fd[idx] = (lp - lm) / (2 * h)
        assert np.allclose(g[k].reshape(fd.shape), fd, rtol=1e-4, atol=1e-7), k
    fdx = np.zeros_like(x)
    for idx in np.ndindex(x.shape):
        xx = x.copy(); xx[idx] += h; lp = L(p, xx); xx[idx] -= 2 * h; lm = L(p, xx)
        fdx[idx] = (lp - lm) / (2 * h)
    assert np.allclose(dx, fdx, rtol=1e-4, atol=1e-7)


def test_decoder_finite_differences():
    # the decoder is smooth given fixed counts: FD on Wd and bd of sum(g_a * a)
    rng = np.random.default_rng(12)
    shp = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5)
    p = sg.randomize_actor(shp, rng, scale=2.5)
    s = rng.uniform(-1, 1, size=(6, 3)).astype(np.float32)
    g_a = rng.standard_normal((6, 2))
    a, tape = oracle.actor_forward(p, shp, s)
    gr = oracle.actor_backward(p, shp, tape, g_a)
    O3 = tape["O"][2]
    h = 1e-6
    for k in ("Wd", "bd"):
        base = p[k].astype(np.float64)
        for idx in np.ndindex(base.shape):
            pl = base.copy(); pl[idx] += h
            mi = base.copy(); mi[idx] -= h
            args = lambda v: (v, p["bd"]) if k == "Wd" else (p["Wd"], v)
            lp = (oracle.decode(O3, *args(pl), 5)[0] * g_a).sum()
            lm = (oracle.decode(O3, *args(mi), 5)[0] * g_a).sum()
            assert abs(gr[k][idx] - (lp - lm) / (2 * h)) <= 1e-6 * max(1, abs(gr[k][idx]))


# ------------------------------------------------------------------ TD3 / Adam / Polyak arithmetic
def _const_critic(in_dim, q):
    return {"W1": np.zeros((4, in_dim)), "b1": np.zeros(4), "W2": np.zeros((4, 4)), "b2": np.zeros(4),
            "W3": np.zeros((1, 4)), "b3": np.array([q])}


def _small_td3(rng, precision="fp32"):
    shp = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5, precision=precision)
    cs = sg.CriticShape(5, 16, 16, precision=precision)
    return shp, cs


def test_td3_target_arithmetic():
    rng = np.random.default_rng(13)
    shp, cs = _small_td3(rng)
    actor = sg.actor_params(shp, rng)
    st = oracle.init_state(actor, _const_critic(5, 0.0), _const_critic(5, 0.0))
    st["c_t"] = [_const_critic(5, 2.0), _const_critic(5, 3.0)]
    batch = sg.replay_batch(rng, 4, 3, 2)
    batch["r"][:] = 1.0; batch["d"][:] = [0, 1, 0, 1]
    hp = sg.TD3Hyper()
    _, info = oracle.td3_update(st, shp, cs, hp, batch, np.zeros((4, 2)), 1)
    assert np.allclose(info["y"], [2.98, 1.0, 2.98, 1.0], rtol=0, atol=1e-15)
    # sigma~ = c = 0 -> a~ = pi'(s')
    a2, _ = oracle.actor_forward(st["actor_t"], shp, batch["s2"])
    hp0 = sg.TD3Hyper(policy_noise=0.0, noise_clip=0.0)
    _, info0 = oracle.td3_update(st, shp, cs, hp0, batch, np.full((4, 2), 0.3), 1)
    assert np.array_equal(info0["a_target"], np.clip(a2, -1, 1))
    assert np.all(info["y"][[0, 2]] <= 1 + 0.99 * 3.0)   # min(Q1', Q2') <= each


def test_td3_lr_zero_and_delay():
    rng = np.random.default_rng(14)
    shp, cs = _small_td3(rng)
    st = oracle.init_state(sg.actor_params(shp, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
    hp0 = sg.TD3Hyper(lr_actor=0.0, lr_critic=0.0)
    b = sg.replay_batch(rng, 8, 3, 2)
    eps = sg.target_noise(rng, 8, 2)
    s1, _ = oracle.td3_update(st, shp, cs, hp0, b, eps, 1)
    s2, _ = oracle.td3_update(s1, shp, cs, hp0, b, eps, 2)
    for a_, b_ in ((st["actor"], s2["actor"]), (st["c"][0], s2["c"][0]), (st["c"][1], s2["c"][1])):
        assert all(np.array_equal(a_[k], b_[k]) for k in a_)
    hp = sg.TD3Hyper()
    s1, i1 = oracle.td3_update(st, shp, cs, hp, b, eps, 1)
    assert "actor_loss" not in i1
    assert all(np.array_equal(st["actor"][k], s1["actor"][k]) for k in st["actor"])
    assert all(np.array_equal(st["c_t"][0][k], s1["c_t"][0][k]) for k in st["c_t"][0])
    assert any(not np.array_equal(st["c"][0][k], s1["c"][0][k]) for k in st["c"][0])
    s2, i2 = oracle.td3_update(s1, shp, cs, hp, b, eps, 2)
    assert "actor_loss" in i2
    assert any(not np.array_equal(s1["actor"][k], s2["actor"][k]) for k in s1["actor"])
    assert any(not np.array_equal(s1["c_t"][1][k], s2["c_t"][1][k]) for k in s1["c_t"][1])


def test_polyak_pins():
    assert oracle.polyak(np.array([0.0]), np.array([1.0]), 0.005)[0] == 0.005
    x = np.random.default_rng(0).standard_normal(50)
    y = np.random.default_rng(1).standard_normal(50)
    assert np.array_equal(oracle.polyak(y, x, 1.0), x)
    assert np.allclose(oracle.polyak(x, x, 0.37), x, rtol=4e-16, atol=0)   # fixed point (to rounding)
    d0 = np.abs(y - x)
    y1 = oracle.polyak(y, x, 0.005)
    assert np.allclose(np.abs(y1 - x), 0.995 * d0, rtol=1e-12)


def test_adam_step1_pin():
    p, m, v = oracle.adam_update(np.array([1.0]), np.array([0.5]), 0.0, 0.0, 1, 1e-3)
    assert abs(p[0] - 0.99900000002) < 1e-14
    g = np.array([3e-3, -2.0, 1e-9, 0.0])
    p1, _, _ = oracle.adam_update(np.zeros(4), g, 0.0, 0.0, 1, 1e-3)
    assert np.allclose(-p1, 1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0)


# ------------------------------------------------------------------ data-parallel equivalence
def test_data_parallel_mean_of_shards():
    rng = np.random.default_rng(15)
    cs = sg.CriticShape(7, 16, 16, precision="fp32")
    p = {k: v.astype(np.float64) for k, v in sg.critic_params(cs, rng).items()}
    x = rng.standard_normal((32, 7)); y = rng.standard_normal(32)
    def grad(xx, yy):
        Q, c = oracle.critic_forward(p, xx)
        return oracle.critic_backward(p, c, 2 * (Q - yy) / len(yy))[0]
    full = grad(x, y)
    shards = [grad(x[i::4], y[i::4]) for i in range(4)]
    for k in full:
        assert np.allclose(full[k], sum(s[k] for s in shards) / 4, rtol=1e-12, atol=1e-15)
    # actor: per-sample independence -> shard gradients of g_a/B average to the full one
    shp = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5)
    pa = sg.randomize_actor(shp, rng, scale=2.5)
    s = rng.uniform(-1, 1, size=(16, 3)).astype(np.float32)
    g_a = rng.standard_normal((16, 2))
    def agrad(ss, gg):
        a, tape = oracle.actor_forward(pa, shp, ss)
        return oracle.actor_backward(pa, shp, tape, gg / len(gg))
    fa = agrad(s, g_a)
    sh = [agrad(s[i * 4:(i + 1) * 4], g_a[i * 4:(i + 1) * 4]) for i in range(4)]
    for k in fa:
        assert np.allclose(fa[k], sum(x_[k] for x_ in sh) / 4, rtol=1e-10, atol=1e-14), k


# ------------------------------------------------------------------ invariants
def test_actor_invariants_cfg0_shape():
    shp, _, B = sg.preset("cfg0")
    rng = np.random.default_rng(0)
    p = sg.actor_params(shp, rng)
    s = sg.observations(rng, 32, shp.obs_dim)
    a, tape = oracle.actor_forward(p, shp, s)
    for O in [tape["O0"]] + tape["O"]:
        assert set(np.unique(O)).issubset({0, 1})
    cnt = oracle.counts(tape)
    assert cnt.max() <= shp.T and np.all(tape["fr"] >= 0) and np.all(tape["fr"] <= 1)
    assert np.all(np.abs(a) < 1)
    a2, _ = oracle.actor_forward(p, shp, s)
    assert np.array_equal(a, a2)                                   # deterministic
    # workload structure: He-uniform gives non-degenerate densities
    dens = [float(O.mean()) for O in tape["O"]]
    assert 0.05 < dens[0] < 0.5 and 0.05 < dens[2] < 0.6, dens


def test_grad_scaler_state_machine():
    """GradScaler rule (PyTorch GradScaler): hand-worked sequences."""
    st = (65536.0, 0)
    st, took = oracle.amp_step(st, True, interval=3)
    assert took and st == (65536.0, 1)
    st, took = oracle.amp_step(st, False, interval=3)        # overflow: skip, back off, reset
    assert not took and st == (32768.0, 0)
    for _ in range(2):
        st, took = oracle.amp_step(st, True, interval=3)
    assert st == (32768.0, 2)
    st, took = oracle.amp_step(st, True, interval=3)         # third finite step in a row: grow
    assert took and st == (65536.0, 0)
    # unscaling by a power-of-two scale is exact; non-finite detection
    g = np.array([1.5, -3.0e-20, 7.0], np.float32)
    assert np.array_equal(oracle.unscale(g * np.float32(65536.0), 65536.0), g)
    assert oracle.all_finite(g) and not oracle.all_finite(np.array([1.0, np.inf], np.float32))
    assert not oracle.all_finite(np.array([np.nan], np.float32))


def test_fp16_rne_laws():
    """fp16 operand rounding (PAPER.md:164 FP16 AMP): IEEE binary16 round-to-nearest-even from fp32."""
    from oracle.numerics import fp16
    assert fp16(1.0 + 2.0 ** -11) == 1.0                 # tie -> even
    assert fp16(1.0 + 3 * 2.0 ** -11) == 1.0 + 2.0 ** -9  # tie -> even (upwards)
    assert fp16(2.0 ** -25) == 0.0                       # half the smallest subnormal -> 0 (even)
    assert fp16(3 * 2.0 ** -25) == 2.0 ** -23            # tie between 2^-24 and 2^-23 -> even
    assert np.isinf(fp16(65520.0)) and fp16(65504.0) == 65504.0
    x = np.random.default_rng(0).normal(0, 10, 1000)
    r = fp16(x)
    assert np.array_equal(fp16(r), r)                    # idempotent
    assert np.all(np.abs(r - x) <= np.maximum(np.abs(x) * 2.0 ** -11, 2.0 ** -25))


# ------------------------------------------------------------------ R20: where the bf16 roundings sit
def _r20_tape():
    """A hand-made tape (the backward is a function of the tape): T = 2, one neuron
    per layer, every hidden/output neuron fires at both steps with V = (0.6, 0.9) (inside the window,
    h = 1), encoder spikes (0, 1) from A = RN32(exp(-1/2)) (s = 1, mu = 0, sigma = 1), a = 0.5, fr = 1."""
    V = np.array([[[0.6]], [[0.9]]])
    O = np.ones((2, 1, 1), np.uint8)
    A = np.array([[np.float32(np.exp(-0.5))]], np.float32)
    tape = dict(A=A, O0=np.array([[[0]], [[1]]], np.uint8), O=[O, O, O], V=[V, V, V],
                a=np.array([[0.5]]), fr=np.array([[1.0]]), s=np.array([[1.0]], np.float32))
    w = 1.0 + 2.0 ** -7 + 2.0 ** -9                      # exact in fp32, not in bf16
    p = dict(mu=np.zeros((1, 1), np.float32), sigma=np.ones((1, 1), np.float32),
             W1=np.full((1, 1), 0.75, np.float32), W2=np.full((1, 1), 0.7, np.float32),
             W3=np.full((1, 1), 0.6, np.float32), Wd=np.full((1, 1), w, np.float32), bd=np.zeros(1, np.float32))
    return p, tape


def test_r20_actor_rounding_points_hand_worked():
    """DESIGN.md R20 for the actor backward, by hand (g_a = 1, d_c = 0.5, rho = 0; o = 1 everywhere so
    the d_v term vanishes):
      g_pre = 1 (1 - 0.5^2) = 0.75; dWd = dbd = 0.75 (fr = 1; the decoder is never rounded)
      g_o3 = 0.75 w / T = 0.375 w;  G3 = (g + d_c g, g) = (0.5625 w, 0.375 w) = (0.5679931640625, 0.378662109375)
      bf16: RN(G3) = (0.56640625, 0.37890625)  [1.0010001|01101b x 2^-1 down; 1.1000001|111b x 2^-2 up]
      dW3 = sum_t RN(G3_t) o2_t = 0.9453125        (unrounded G3 would give 0.9466552734375)
      RN(W3 = 0.6f) = 0.6015625;  g_o2 = RN(G3) RN(W3) = (0.340728759765625, 0.227935791015625)
      G2 = (g_o2[1] + 0.5 g_o2[2], g_o2[2]) = (0.4546966552734375, 0.227935791015625) -> RN (0.455078125, 0.2275390625)
      dW2 = 0.6826171875;  RN(W2 = 0.7f) = 0.69921875;  g_o1 = RN(G2) RN(W2)
      G1 = (0.3977489471435547, 0.15909957885742188) -> RN (0.3984375, 0.1591796875)
      dW1 = RN(G1_2) o0_2 = 0.1591796875   (o0 = (0, 1))
      encoder: RN(sum_t G1) = RN(0.5568485260009766) = 0.55859375 -- the SUM is rounded once (rounding
      each G1_t first would give 0.5576171875); dL/dA = 0.55859375 RN(W1 = 0.75) = 0.4189453125;
      dmu = dL/dA A (s - mu) / sigma^2 = 0.4189453125 RN32(exp(-1/2)) = dsigma (s - mu = sigma = 1)."""
    p, tape = _r20_tape()
    g = oracle.actor_backward(p, cfg_ns(T=2, precision="bf16"), tape, np.array([[1.0]]))
    A = float(np.float32(np.exp(-0.5)))
    assert g["Wd"][0, 0] == 0.75 and g["bd"][0] == 0.75
    assert g["W3"][0, 0] == 0.9453125
    assert g["W2"][0, 0] == 0.6826171875
    assert g["W1"][0, 0] == 0.1591796875
    assert g["mu"][0, 0] == 0.4189453125 * A and g["sigma"][0, 0] == 0.4189453125 * A
    # fp32 mode: nothing rounded; dW3 = 0.9375 w exactly
    g32 = oracle.actor_backward(p, cfg_ns(T=2, precision="fp32"), tape, np.array([[1.0]]))
    assert g32["W3"][0, 0] == 0.9375 * (1.0 + 2.0 ** -7 + 2.0 ** -9)


def test_r20_critic_rounding_points_hand_worked():
    """DESIGN.md R20 for the critic, by hand: in = 2, one hidden unit per layer, x = [1 + 2^-9, 0.5],
    W1 = [1, 1], W2 = w = 1 + 2^-7 + 2^-9, W3 = 1, biases 0, dL/dQ = 1 + 2^-9.
      RN(x) = [1, 0.5] (2^-9 < half an ulp) -> z1 = 1.5 = h1;  RN(w) = 1.0078125;  z2 = 1.51171875
      h2 = RN(z2) = 1.515625 (65.5/128: tie to even 66);  Q = 1.515625
      dh2 = dQ W3 = 1 + 2^-9 -> dz2 = RN(.) = 1;  dz1 = RN(dz2 RN(w)) = 1.0078125;  dx = dz1 RN(W1)
      dW3 = dQ h2 = 1.518585205078125;  db3 = dQ;  dW2 = dz2 h1 = 1.5;  db2 = 1
      dW1 = dz1 RN(x) = [1.0078125, 0.50390625];  db1 = 1.0078125."""
    w = 1.0 + 2.0 ** -7 + 2.0 ** -9
    p = dict(W1=np.ones((1, 2), np.float32), b1=np.zeros(1, np.float32), W2=np.full((1, 1), w, np.float32),
             b2=np.zeros(1, np.float32), W3=np.ones((1, 1), np.float32), b3=np.zeros(1, np.float32))
    x = np.array([[1.0 + 2.0 ** -9, 0.5]])
    q, cache = oracle.critic_forward(p, x, "bf16")
    assert q[0] == 1.515625
    dQ = 1.0 + 2.0 ** -9
    g, dx = oracle.critic_backward(p, cache, np.array([dQ]), "bf16")
    assert g["W3"][0, 0] == 1.518585205078125 and g["b3"][0] == dQ
    assert g["W2"][0, 0] == 1.5 and g["b2"][0] == 1.0
    assert np.array_equal(g["W1"], [[1.0078125, 0.50390625]]) and g["b1"][0] == 1.0078125
    assert np.array_equal(dx, [[1.0078125, 1.0078125]])
    # fp32 mode: x kept, Q = (1 + 2^-9 + 0.5) w
    q32, _ = oracle.critic_forward(p, x, "fp32")
    assert q32[0] == (1.5 + 2.0 ** -9) * w


def test_encoder_exemption_condition():
    """The parity protocol's encoder exemption (C-4 step 2) holds only within 2 ulp64 of an fp32
    rounding midpoint."""
    from tests._parity import near_fp32_midpoint
    mid = 1.0 + 2.0 ** -24                                   # halfway between 1 and 1 + 2^-23
    u = 2.0 ** -52
    vals = np.array([mid, mid + 2 * u, mid - 2 * u, mid + 3 * u, 1.0, 0.75 + 2.0 ** -25, 0.6065306597126334])
    assert near_fp32_midpoint(vals).tolist() == [True, True, True, False, False, True, False]
