"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical seeded inputs.
Tolerances (north_star): encoder spikes bit-exact; fp32 actions
1e-4 relative, spike disagreement <= 1e-5 of spikes and only within 1e-5 of V_th; bf16 actions
2e-2 absolute, gradients 1e-2 relative L2 (fp32 mode: 1e-4)."""
import numpy as np
import pytest

import oracle
import synthgen as sg
from tests._parity import run_gpu_actor, check_actor, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _inputs(shape, B, seed=0):
    rng = np.random.default_rng(seed)
    p = sg.actor_params(shape, rng)
    s = sg.observations(rng, B, shape.obs_dim)
    g = sg.action_grads(rng, B, shape.act_dim)
    return p, s, g


# ------------------------------------------------------------------ encoder (bit-exact, every config shape)
@pytest.mark.parametrize("name,B", [("cfg0", 100), ("cfg1", 256), ("cfg2", 512), ("cfg3s", 100), ("cfg3L", 1024),
                                    ("cfg4", 256)])
def test_encoder_bit_exact(name, B):
    shape, _, _ = sg.preset(name)
    p, s, _ = _inputs(shape, B, seed=1)
    gpu = run_gpu_actor(shape, B, p, s, None, engine="simt")
    from tests._parity import check_encoder
    assert check_encoder(gpu, shape, p, s) == 0


def test_encoder_edge_values():
    """s exactly on mu (A = 1 -> fires every step), far tails (A underflows / subnormal)."""
    shape = sg.ActorShape(1, 1, pop_enc=10, pop_dec=2, n1=32, n2=32, T=5, precision="fp32")
    rng = np.random.default_rng(0)
    p = sg.actor_params(shape, rng)
    s = np.array([[-3.0], [-1.0], [1.0], [0.3333333432674408], [5.0], [-5.0], [0.1], [0.2], [-0.5], [2.9],
                  [1e-30], [4.99]], np.float32)
    gpu = run_gpu_actor(shape, len(s), p, s, None, engine="simt")
    from tests._parity import check_encoder
    assert check_encoder(gpu, shape, p, s) == 0


def test_encoder_quotient_stress():
    """A = RN32(exp(-(s-mu)^2 / (2 sigma^2))) bit-exact over a wide spread of sigma (log-uniform
    1e-3..30, learnable: DESIGN.md R12) and s (N(0, 3^2)): pins the kernel's reciprocal-based
    correctly rounded quotient against the oracle's IEEE division."""
    shape = sg.ActorShape(3, 2, pop_enc=64, pop_dec=4, n1=32, n2=32, T=16, precision="bf16")
    rng = np.random.default_rng(11)
    p = sg.actor_params(shape, rng)
    p["sigma"] = np.exp(rng.uniform(np.log(1e-3), np.log(30.0), p["sigma"].shape)).astype(np.float32)
    p["mu"] = rng.normal(0, 3, p["mu"].shape).astype(np.float32)
    s = rng.normal(0, 3, (2048, 3)).astype(np.float32)
    gpu = run_gpu_actor(shape, 2048, p, s, None, engine="simt")
    from tests._parity import check_encoder
    assert check_encoder(gpu, shape, p, s) == 0


@pytest.mark.parametrize("case", ["cfg1", "cfg3L", "cfg4_512", "cfg0", "T7", "T33", "stress"])
def test_inference_forward_spikes_only(case):
    """The inference-only forward (tape == NULL; TD3's target actor) skips the stimulation plane and
    forms the exact A only where the fp32 screen z32 <= zskip says a spike is possible
    (enc_fwd_kernel SPK): its spike / window planes, counts and actions equal the recording
    forward's bit for bit, and its encoder spikes the oracle's — also over the wide sigma / mu
    spread of the quotient stress case, where the screen's margins are tightest."""
    import torch
    import paper_2502_17496_b200 as pk
    from tests._parity import check_encoder
    engine = "auto"
    if case == "stress":
        shape = sg.ActorShape(3, 2, pop_enc=64, pop_dec=4, n1=32, n2=32, T=16, precision="bf16")
        rng = np.random.default_rng(12)
        p = sg.actor_params(shape, rng)
        p["sigma"] = np.exp(rng.uniform(np.log(1e-3), np.log(30.0), p["sigma"].shape)).astype(np.float32)
        p["mu"] = rng.normal(0, 3, p["mu"].shape).astype(np.float32)
        B = 2048
        s = rng.normal(0, 3, (B, 3)).astype(np.float32)
        engine = "simt"
    else:
        name, B = {"cfg1": ("cfg1", None), "cfg3L": ("cfg3L", 4096), "cfg4_512": ("cfg4", 512), "cfg0": ("cfg0", None),
                   "T7": ("cfg2", 96), "T33": ("cfg2", 45)}[case]
        shape, _, B0 = sg.preset(name)
        B = B or B0
        if case == "T7":
            shape, engine = sg.with_(shape, T=7), "simt"
        if case == "T33":
            shape, engine = sg.with_(shape, T=33), "simt"
        p, s, _ = _inputs(shape, B, seed=21)
    actor = pk.SpikingActor(pk.actor_cfg_from(shape, engine=engine), B)
    actor.load(p)
    obs = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    a_rec = actor.forward(obs).clone()
    sp_rec = actor.spikes()
    cnt_rec = actor.tape_view()["counts"].clone()
    a_inf = actor.forward(obs, record=False).clone()
    tv = actor.inference_tape_view()
    sp_inf = pk.tape_spikes(actor.cfg, tv)
    torch.cuda.synchronize()
    assert torch.equal(a_rec, a_inf)
    assert torch.equal(cnt_rec, tv["counts"])
    for k in sp_rec:
        assert np.array_equal(sp_rec[k], sp_inf[k]), k
    gpu = dict(sp=sp_inf, A=None)
    assert check_encoder(gpu, shape, p, s, a_stored=False) == 0


@pytest.mark.parametrize("T,B,N", [(5, 37, 45), (16, 64, 256), (7, 3, 33), (33, 5, 70)])
def test_lif_scan_ablation(T, B, N):
    """The standalone forward-scan ablation kernel (spikerl_lif_scan_forward) against
    the oracle's LIF layer (north_star equations), teacher forced on the kernel's own
    reset decisions: a spike or window bit may differ only within 1e-5 of V_th or of a window edge
    (the kernel scans the fp32-rounded currents, the oracle the fp64 ones)."""
    import torch
    import paper_2502_17496_b200 as pk
    shape = sg.preset("cfg1")[0]
    rng = np.random.default_rng(T * 1000 + N)
    K = 40
    o_in = (rng.random((T, B, K)) < 0.3).astype(np.uint8)
    Wt = rng.normal(0, 0.6, (N, K))
    _, _, I = oracle.lif_layer_forward(o_in, Wt, shape.d_c, shape.d_v, shape.v_th)
    W = (N + 31) // 32
    Id = torch.from_numpy(I.astype(np.float32)).cuda().contiguous()
    bits = torch.zeros(T, B, W, dtype=torch.int32, device="cuda")
    mask = torch.zeros(T, B, W, dtype=torch.int32, device="cuda")
    lib = pk.lib()
    rc = lib.spikerl_lif_scan_forward(Id.data_ptr(), T, B, N, shape.d_c, shape.d_v, shape.v_th, shape.surr_window,
                                      bits.data_ptr(), mask.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
    torch.cuda.synchronize()
    O = pk.unpack_bits(bits, N)
    H = pk.unpack_bits(mask, N)
    V, O_ref, _ = oracle.lif_layer_forward(o_in, Wt, shape.d_c, shape.d_v, shape.v_th, forced_o=O)
    near = np.abs(V - shape.v_th) < 1e-5
    assert not np.any((O.astype(bool) != O_ref.astype(bool)) & ~near)
    h_ref = np.abs(V - shape.v_th) < shape.surr_window
    near_h = np.minimum(np.abs(V - (shape.v_th - shape.surr_window)), np.abs(V - (shape.v_th + shape.surr_window))) < 1e-5
    assert not np.any((H.astype(bool) != h_ref) & ~near_h)
    assert O.any() and (~O.astype(bool)).any()


@pytest.mark.parametrize("T", [7, 32, 33, 70])
def test_encoder_timesteps(T):
    """Unrolled (T in the compiled set) and runtime-T (chunks of 32 steps) encoder variants."""
    shape = sg.with_(sg.preset("cfg2")[0], T=T)
    p, s, _ = _inputs(shape, 45, seed=T)
    gpu = run_gpu_actor(shape, 45, p, s, None, engine="simt")
    from tests._parity import check_encoder
    assert check_encoder(gpu, shape, p, s) == 0


# ------------------------------------------------------------------ fp32 actor (configs[0])
def test_actor_fp32_cfg0():
    shape, _, B = sg.preset("cfg0")
    p, s, g = _inputs(shape, B)
    gpu = run_gpu_actor(shape, B, p, s, g)
    st = check_actor(gpu, shape, p, s, g)
    assert st["free_flips"] == [0, 0, 0], st


@pytest.mark.parametrize("B", [1, 7, 33, 129])
def test_actor_fp32_ragged_batches(B):
    shape, _, _ = sg.preset("cfg0")
    p, s, g = _inputs(shape, B, seed=B)
    check_actor(run_gpu_actor(shape, B, p, s, g), shape, p, s, g)


@pytest.mark.parametrize("T", [1, 2, 16, 31])
def test_actor_fp32_timesteps(T):
    shape = sg.with_(sg.preset("cfg0")[0], T=T)
    p, s, g = _inputs(shape, 64, seed=T)
    check_actor(run_gpu_actor(shape, 64, p, s, g), shape, p, s, g)


def test_actor_fp32_odd_widths():
    # widths that are not multiples of 32/128: padding must not change results (R28)
    shape = sg.ActorShape(5, 3, pop_enc=7, pop_dec=9, n1=45, n2=161, T=5, precision="fp32")
    p, s, g = _inputs(shape, 50, seed=3)
    check_actor(run_gpu_actor(shape, 50, p, s, g), shape, p, s, g)


def test_zero_decoder_and_zero_network():
    shape, _, _ = sg.preset("cfg0")
    p, s, g = _inputs(shape, 32)
    p["Wd"] = np.zeros_like(p["Wd"]); p["bd"] = np.linspace(-0.5, 0.5, shape.act_dim).astype(np.float32)
    gpu = run_gpu_actor(shape, 32, p, s, g)
    assert np.allclose(gpu["a"], np.tanh(p["bd"].astype(np.float64))[None], atol=1e-6)
    for k in ("mu", "sigma", "W1", "W2", "W3"):
        assert np.all(gpu["grads"][k] == 0), k
    check_actor(gpu, shape, p, s, g)
    for k in ("W1", "W2", "W3", "Wd", "bd"):
        p[k] = np.zeros_like(p[k])
    gpu = run_gpu_actor(shape, 32, p, s, np.zeros_like(g))
    assert np.all(gpu["a"] == 0) and all(np.all(v == 0) for v in gpu["grads"].values())


# ------------------------------------------------------------------ bf16 actor (configs[1..4] shapes)
@pytest.mark.parametrize("name,B,engine", [("cfg1", 256, "auto"), ("cfg2", 512, "auto"), ("cfg3s", 100, "auto"),
                                           ("cfg3L", 1024, "auto"), ("cfg3L", 4096, "auto"), ("cfg1", 256, "simt"),
                                           ("cfg3L", 300, "simt")])
def test_actor_bf16(name, B, engine):
    """configs[1..3] shapes at their per-rank batches; configs[3] at B = 4096 is the launch configuration
    of the bench's TD3 throughput line (its forward layers run the Bt = 32 batch tiles)."""
    shape, _, _ = sg.preset(name)
    p, s, g = _inputs(shape, B, seed=2)
    st = check_actor(run_gpu_actor(shape, B, p, s, g, engine=engine), shape, p, s, g)
    print(name, B, engine, st)


@pytest.mark.parametrize("T,B", [(1, 17), (2, 1), (3, 50), (5, 1), (8, 33), (16, 19), (24, 40)])
def test_actor_bf16_tcgen05_edges(T, B):
    """tcgen05 engine on odd widths (padding rows/cols), ragged and tiny batches and every
    batch-tile shape the tile chooser can pick (T*Bt in {16..256})."""
    shape = sg.ActorShape(5, 3, pop_enc=7, pop_dec=9, n1=45, n2=161, T=T, precision="bf16")
    p, s, g = _inputs(shape, B, seed=10 + T)
    check_actor(run_gpu_actor(shape, B, p, s, g, engine="tcgen05"), shape, p, s, g)


@pytest.mark.parametrize("name,B", [("cfg2", 96), ("cfg1", 256), ("cfg1", 37)])
def test_engines_agree_on_spikes(name, B):
    """tcgen05 and SIMT engines compute the same currents up to summation order: their spike
    planes agree except for decisions within 1e-5 of the threshold (none expected here)."""
    shape, _, _ = sg.preset(name)
    p, s, g = _inputs(shape, B, seed=21)
    a = run_gpu_actor(shape, B, p, s, g, engine="tcgen05")
    b = run_gpu_actor(shape, B, p, s, g, engine="simt")
    for l in range(4):
        assert np.array_equal(a["sp"][f"o{l}"], b["sp"][f"o{l}"]), l
    for k in a["grads"]:
        assert rel_l2(a["grads"][k], b["grads"][k]) <= 5e-3, k


def test_actor_bf16_cfg4_shape_subsample():
    """configs[4] widths (1024-1024, T=16) on a 64-row sample (teacher forced)."""
    shape, _, _ = sg.preset("cfg4")
    p, s, g = _inputs(shape, 64, seed=4)
    st = check_actor(run_gpu_actor(shape, 64, p, s, g), shape, p, s, g)
    print(st)


def test_actor_bf16_cfg4_full_batch():
    """configs[4] at its full batch (65 536 rows: the launch configuration bench.py times).
    Forward: the oracle re-runs 96 sampled rows teacher forced (spikes, masks, actions, encoder).
    Backward: every row's G_l is independent of the batch it runs in, so the full-batch gradient
    (one split-K plan, 2048 N tiles per layer) must equal the fp64 sum of the gradients of four
    16 384-row chunks (other plans); the 64-row oracle check above pins the per-row backward."""
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, Bg = sg.preset("cfg4")
    p, s, g = _inputs(shape, Bg, seed=7)
    actor = pk.SpikingActor(pk.actor_cfg_from(shape), Bg)
    actor.load(p)
    obs = torch.from_numpy(s).cuda()
    ga = torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda()
    a = actor.forward(obs)
    full = actor.backward(obs, ga).double().cpu()
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(3).choice(Bg, 96, replace=False))
    rt = torch.from_numpy(rows).cuda()
    v = actor.tape_view()
    N = [shape.obs_dim * shape.pop_enc, shape.n1, shape.n2, shape.act_dim * shape.pop_dec]
    sp = {f"o{l}": pk.unpack_bits(v[f"bits{l}"][:, rt, :], N[l]) for l in range(4)}
    sp.update({f"h{l}": pk.unpack_bits(v[f"mask{l}"][:, rt, :], N[l]) for l in (1, 2, 3)})
    gpu = dict(a=a[rt].cpu().numpy().astype(np.float64), grads=None, sp=sp, A=v["A"][rt].cpu().numpy(),
               counts=v["counts"][rt].cpu().numpy())
    print(check_actor(gpu, shape, p, s[rows], None))
    del actor, v
    Bc = Bg // 4
    chunk = pk.SpikingActor(pk.actor_cfg_from(shape), Bc)
    chunk.load(p)
    tot = torch.zeros_like(full)
    for c in range(4):
        tot += _fwd_bwd(chunk, obs[c * Bc:(c + 1) * Bc], ga[c * Bc:(c + 1) * Bc])
    gf, gt = pk.unpack_actor(chunk.cfg, full.float()), pk.unpack_actor(chunk.cfg, tot.float())
    for k in gf:
        e = rel_l2(gf[k], gt[k])
        assert e <= 1e-4, (k, e)


def _fwd_bwd(actor, obs, ga):
    import torch
    actor.forward(obs)
    out = actor.backward(obs, ga).double().cpu()
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("B", [100, 257])
def test_neuron_major_planes_are_transposes(B):
    """tcgen05 engine: the quad-major spike/mask copies read by the fused dX epilogue hold
    exactly the transposed bits of the batch-major planes (bit-exact, ragged batch)."""
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, _ = sg.preset("cfg1")
    p, s, _ = _inputs(shape, B)
    actor = pk.SpikingActor(pk.actor_cfg_from(shape, engine="tcgen05"), B)
    actor.load(p)
    actor.forward(torch.from_numpy(s).cuda())
    torch.cuda.synchronize()
    v = actor.tape_view()
    for l in (1, 2):
        for a, bname in ((f"bits{l}", f"bitsT{l}"), (f"mask{l}", f"maskT{l}")):
            bm = pk.unpack_bits(v[a], v[a].shape[-1] * 32)              # [T][B][P]
            raw = v[bname].cpu().numpy()                                # [Q][P][tpad/2] bytes
            bits = np.unpackbits(raw[..., None], axis=-1, bitorder="little")   # [Q][P][tpad/2][8]
            Q, P = raw.shape[0], raw.shape[1]
            bits = bits.reshape(Q, P, raw.shape[2] * 2, 4)               # nibble s = step s
            nm = bits.transpose(2, 1, 0, 3).reshape(raw.shape[2] * 2, P, -1)  # [tpad][P][Q*4]
            T = shape.T
            assert np.array_equal(nm[:T, :, :B], bm.transpose(0, 2, 1)), (l, a)
            assert not nm[:T, :, B:].any() and not nm[T:].any()


def test_backward_rejects_foreign_tape():
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, _ = sg.preset("cfg0")
    p, s, g = _inputs(shape, 8)
    a1 = pk.SpikingActor(pk.actor_cfg_from(shape), 8)
    a1.load(p)
    obs = torch.from_numpy(s).cuda()
    with pytest.raises(pk.SpikeRLError) as e:
        a1.backward(obs, torch.from_numpy(g).cuda())       # no forward yet -> tape not stamped
    assert e.value.status == 3
    a1.forward(obs)
    a2 = pk.SpikingActor(pk.actor_cfg_from(sg.with_(shape, T=4)), 8)
    a2.load(p)
    a2.tape = a1.tape
    with pytest.raises(pk.SpikeRLError):
        a2.backward(obs, torch.from_numpy(g).cuda())


def test_forward_deterministic_and_accumulate():
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, _ = sg.preset("cfg1")
    p, s, g = _inputs(shape, 64)
    act = pk.SpikingActor(pk.actor_cfg_from(shape), 64)
    act.load(p)
    obs = torch.from_numpy(s).cuda(); ga = torch.from_numpy(g).cuda()
    a1 = act.forward(obs).clone(); g1 = act.backward(obs, ga).clone()
    a2 = act.forward(obs).clone(); g2 = act.backward(obs, ga).clone()
    assert torch.equal(a1, a2) and torch.equal(g1, g2)           # bitwise run-to-run
    g3 = act.backward(obs, ga, accumulate=True).clone()
    assert torch.allclose(g3, 2 * g1, rtol=1e-6, atol=0)


# ------------------------------------------------------------------ reset-gate gradient (rho = 1)
@pytest.mark.parametrize("name,B,prec,engine,T", [("cfg0", 100, "fp32", "auto", 5), ("cfg1", 256, "bf16", "auto", 5),
                                                 ("cfg1", 256, "bf16", "simt", 5), ("cfg3L", 1024, "bf16", "auto", 5),
                                                 ("cfg3L", 4096, "bf16", "auto", 5), ("cfg4", 64, "bf16", "auto", 16),
                                                 ("odd", 33, "bf16", "auto", 16), ("odd", 19, "fp32", "auto", 7)])
def test_actor_reset_grad(name, B, prec, engine, T):
    """SPEC.md:171's variant with the reset gate differentiated (rho = 1, R11): the fp32
    membrane potentials kept in the tape and the reverse scans (SIMT, tcgen05 DX epilogue, output-layer
    scan) against the oracle's rho = 1 BPTT, teacher forced, at the rho = 0 tolerances; the variant
    must matter (the rho = 0 gradient is far from it) and leave the forward unchanged."""
    if name == "odd":
        shape = sg.ActorShape(5, 3, pop_enc=7, pop_dec=9, n1=45, n2=161, T=T, precision=prec)
    else:
        shape = sg.with_(sg.preset(name)[0], precision=prec, T=T)
    p, s, g = _inputs(shape, B, seed=40 + B)
    gpu = run_gpu_actor(shape, B, p, s, g, engine=engine, reset_grad=1)
    st = check_actor(gpu, shape, p, s, g, rho=1.0)
    ref0 = run_gpu_actor(shape, B, p, s, g, engine=engine, reset_grad=0)
    assert np.array_equal(ref0["a"], gpu["a"]) and all(np.array_equal(ref0["sp"][k], gpu["sp"][k]) for k in gpu["sp"])
    assert max(rel_l2(gpu["grads"][k], ref0["grads"][k]) for k in ("W1", "W2", "W3")) > 0.05, "rho had no effect"
    print(name, B, prec, st.get("grad_rel_l2"))


# ------------------------------------------------------------------ critic
@pytest.mark.parametrize("prec,B,S,A", [("fp32", 100, 17, 6), ("bf16", 256, 17, 6), ("bf16", 4096, 17, 6),
                                        ("bf16", 100, 376, 17), ("bf16", 512, 111, 8), ("bf16", 37, 17, 6),
                                        ("bf16", 1040, 376, 17), ("bf16", 4096, 376, 17), ("bf16", 1500, 17, 6),
                                        ("bf16", 1024, 111, 8)])
def test_critic_parity(prec, B, S, A):
    """fp32 SIMT critic, the warp-MMA bf16 critic (B < 2048) and the tcgen05 bf16 critic (B >= 2048:
    configs[3] B = 4096, configs[1] widths at 4096) against the oracle."""
    import torch
    import paper_2502_17496_b200 as pk
    rng = np.random.default_rng(5)
    cs = sg.CriticShape(S + A, precision=prec)
    c1, c2 = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
    for c in (c1, c2):
        for k in ("b1", "b2", "b3"):
            c[k] = rng.uniform(-0.2, 0.2, c[k].shape).astype(np.float32)
    batch = sg.replay_batch(rng, B, S, A)
    y = rng.standard_normal(B).astype(np.float32)
    tc = pk.TwinCritic(pk.critic_cfg(S + A, precision=prec), B)
    tc.load(c1, c2)
    obs = torch.from_numpy(batch["s"]).cuda(); act = torch.from_numpy(batch["a"]).cuda()
    yt = torch.from_numpy(y).cuda()
    ga = torch.zeros(B, A, device="cuda")
    q = tc(obs, act, yt).cpu().numpy()
    grads = tc.grads.cpu().numpy()
    loss = float(tc.loss.cpu())
    tc(obs, act, None, grad_act=ga, act_grad_scale=-1.0 / B)
    ga = ga.cpu().numpy()
    x = np.concatenate([batch["s"], batch["a"]], 1).astype(np.float64)
    tol_q = 1e-4 if prec == "fp32" else 2e-2
    gt = 1e-4 if prec == "fp32" else 1e-2
    lref = 0.0
    P = tc.P
    for i, cp in enumerate((c1, c2)):
        qr, cache = oracle.critic_forward(cp, x, prec)
        assert np.allclose(q[i], qr, rtol=tol_q, atol=tol_q), (i, np.abs(q[i] - qr).max())
        lref += np.mean((qr - y) ** 2)
        gr, _ = oracle.critic_backward(cp, cache, 2 * (qr - y) / B, prec)
        mine = pk.unpack_critic(tc.cfg, grads[i * P:(i + 1) * P])
        for k in gr:
            assert rel_l2(mine[k].reshape(gr[k].shape), gr[k]) <= gt, (i, k)
        if i == 0:
            _, dx = oracle.critic_backward(cp, cache, np.full(B, -1.0 / B), prec, need_param_grads=False)
            assert rel_l2(ga, dx[:, S:]) <= gt
    assert abs(loss - lref) <= gt * abs(lref)


# ------------------------------------------------------------------ Adam / Polyak
def test_adam_and_polyak():
    import torch
    import paper_2502_17496_b200 as pk
    rng = np.random.default_rng(6)
    n = 10007
    p = rng.standard_normal(n).astype(np.float32)
    p[:10] = 0.0005
    pt = torch.from_numpy(p).cuda()
    m = torch.zeros(n, device="cuda"); v = torch.zeros(n, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    pr, mr, vr = p.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(1, 4):
        g = rng.standard_normal(n).astype(np.float32)
        pk.adam(pt, torch.from_numpy(g).cuda(), m, v, cnt, 1e-3, clamp=(0, 10, 1e-3))
        pr, mr, vr = oracle.adam_update(pr, g, mr, vr, t, 1e-3)
        pr[:10] = np.maximum(pr[:10], 1e-3)
    assert int(cnt[0]) == 3 and int(cnt[1]) == 0
    assert np.allclose(pt.cpu().numpy(), pr, rtol=0, atol=1e-6)
    assert np.allclose(m.cpu().numpy(), mr, rtol=1e-5, atol=1e-7)
    assert np.all(pt.cpu().numpy()[:10] >= 1e-3)
    src = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
    tgt = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
    ref = oracle.polyak(tgt.cpu().numpy(), src.cpu().numpy(), 0.005)
    pk.polyak(tgt, src, 0.005)
    assert np.allclose(tgt.cpu().numpy(), ref, rtol=0, atol=1e-6)
    pk.polyak(tgt, src, 1.0)
    assert torch.equal(tgt, src)


# ------------------------------------------------------------------ TD3 update (oracle parity: tests/test_gpu_td3_parity.py)
def test_critic_tcgen05_small_and_ragged_subprocess():
    """The tcgen05 critic forced below its default threshold (SPIKERL_CRITIC_TC=2: B >= 512, a
    subprocess): configs[2] widths at 512, ragged batches whose last 128-row tile ends in a partly
    (1500) or wholly (1450) out-of-bounds TMA box, against the oracle through the same checks."""
    import os, subprocess, sys
    code = (
        "import sys; sys.argv = ['x']\n"
        "import tests.test_gpu_parity as t\n"
        "for args in (('bf16', 512, 111, 8), ('bf16', 1500, 376, 17), ('bf16', 1450, 17, 6)):\n"
        "    t.test_critic_parity(*args)\n"
        "print('tc critic ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, SPIKERL_CRITIC_TC="2", PYTHONPATH=root))
    assert r.returncode == 0 and "tc critic ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("name,B", [("cfg1", 256), ("cfg3L", 4096)])
def test_td3_schedule_independent_subprocess(name, B):
    """The TD3 update-pair DAG's scheduling switches change streams, priorities and launch edges only:
    four update pairs (captured graphs) end in bitwise identical actor / critic / target parameters and
    Adam moments under the default schedule, SPIKERL_TD3_SERIAL=1 (one stream), SPIKERL_TD3_PRIO=0 / 5
    (no / raised launch priority) and SPIKERL_PDL=0 (no programmatic dependent launch)."""
    import os, subprocess, sys
    code = (
        "import hashlib, numpy as np, torch\n"
        "import synthgen as sg, paper_2502_17496_b200 as pk\n"
        f"shape, _, _ = sg.preset({name!r}); B = {B}\n"
        "S, A = shape.obs_dim, shape.act_dim\n"
        "rng = np.random.default_rng(3)\n"
        "cs = sg.CriticShape(S + A, precision='bf16')\n"
        "td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(S + A), pk.td3_cfg(B), pk.replay_fill(4 * B, S, A, seed=4), seed=6)\n"
        "td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))\n"
        "td3.update_pair(1)\n"
        "td3.capture_pair()\n"
        "for _ in range(4): td3.replay_pair()\n"
        "torch.cuda.synchronize()\n"
        "h = hashlib.sha256()\n"
        "for t in (td3.actor, td3.actor_t, td3.critic, td3.critic_t, td3.m_actor, td3.v_actor, td3.m_critic, td3.v_critic):\n"
        "    h.update(t.cpu().numpy().tobytes())\n"
        "print('digest', h.hexdigest())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = {}
    for label, extra in (("default", {}), ("serial", {"SPIKERL_TD3_SERIAL": "1"}), ("prio0", {"SPIKERL_TD3_PRIO": "0"}),
                         ("prio5", {"SPIKERL_TD3_PRIO": "5"}), ("nopdl", {"SPIKERL_PDL": "0"})):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, PYTHONPATH=root, **extra))
        assert r.returncode == 0, (label, r.stdout[-1500:] + r.stderr[-1500:])
        digests[label] = [l for l in r.stdout.splitlines() if l.startswith("digest")][-1]
    assert len(set(digests.values())) == 1, digests


@pytest.mark.parametrize("name,B", [("cfg1", 256), ("cfg1", 200), ("cfg2", 512), ("cfg3s", 100), ("cfg3s", 37)])
def test_td3_fused_critic_matches_separate_launches_subprocess(name, B):
    """The fused small-batch critic launches (the whole critic update, forward to Adam + Polyak, with
    grid barriers; the actor objective's critic pass) are bitwise the separate launches
    (SPIKERL_CRITIC_FUSED=0), the layout-aware critic Adam is bitwise the flat adam_kernel
    (SPIKERL_CRITIC_ADAM_TILED=0), the target decoder inside the target critics' launch bitwise its own
    launch (SPIKERL_CRITIC_DECODE=0): two single updates, then three captured update pairs end in identical
    parameters, targets, Adam moments and step counts, losses and dQ1/da, at several grid sizes."""
    import os, subprocess, sys
    code = (
        "import hashlib, numpy as np, torch\n"
        "import synthgen as sg, paper_2502_17496_b200 as pk\n"
        f"shape, _, _ = sg.preset({name!r}); B = {B}\n"
        "S, A = shape.obs_dim, shape.act_dim\n"
        "rng = np.random.default_rng(5)\n"
        "cs = sg.CriticShape(S + A, precision='bf16')\n"
        "td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(S + A), pk.td3_cfg(B), pk.replay_fill(4 * B, S, A, seed=4), seed=7)\n"
        "td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))\n"
        "h = hashlib.sha256()\n"
        "for k in (1, 2):\n"
        "    td3.update(k)\n"
        "    torch.cuda.synchronize()\n"
        "    h.update(td3.losses.cpu().numpy().tobytes())\n"
        "td3.update_pair(3)\n"
        "td3.capture_pair()\n"
        "for _ in range(3): td3.replay_pair()\n"
        "torch.cuda.synchronize()\n"
        "for t in (td3.actor, td3.actor_t, td3.critic, td3.critic_t, td3.m_actor, td3.v_actor, td3.m_critic,\n"
        "          td3.v_critic, td3.adam_steps, td3.losses, td3.critic_bf16, td3.critic_t_bf16, td3.rng_counter):\n"
        "    h.update(t.cpu().numpy().tobytes())\n"
        "print('digest', h.hexdigest())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = {}
    for label, extra in (("fused", {"SPIKERL_CRITIC_FUSED": "1"}), ("separate", {"SPIKERL_CRITIC_FUSED": "0"}),
                         ("separate_flat_adam", {"SPIKERL_CRITIC_FUSED": "0", "SPIKERL_CRITIC_ADAM_TILED": "0",
                                                 "SPIKERL_CRITIC_ACT_FUSED": "0"}),
                         ("separate_merged_wg", {"SPIKERL_CRITIC_FUSED": "0", "SPIKERL_CRITIC_WG_MERGE": "1"}),
                         ("decoder_launch", {"SPIKERL_CRITIC_DECODE": "0"}),
                         ("fused_g148", {"SPIKERL_CRITIC_FUSED": "1", "SPIKERL_CRITIC_FUSED_G": "148"}),
                         ("fused_gmin", {"SPIKERL_CRITIC_FUSED": "1", "SPIKERL_CRITIC_FUSED_G": "1"})):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, PYTHONPATH=root, **extra))
        assert r.returncode == 0, (label, r.stdout[-1500:] + r.stderr[-1500:])
        digests[label] = [l for l in r.stdout.splitlines() if l.startswith("digest")][-1]
    assert len(set(digests.values())) == 1, digests


@pytest.mark.parametrize("obs,act", [(17, 6), (111, 8)])
def test_td3_bf16_copies_track_masters(obs, act):
    """Adam / Polyak write the bf16 working copies in place (Bf16Views): after several updates they
    must equal, bit for bit, a full refresh of the fp32 masters (padding included)."""
    import torch
    import paper_2502_17496_b200 as pk
    shape = sg.with_(sg.preset("cfg1")[0], obs_dim=obs, act_dim=act)
    replay = pk.replay_fill(5000, obs, act, seed=5)
    rng = np.random.default_rng(9)
    cs = sg.CriticShape(obs + act, precision="bf16")
    td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(obs + act), pk.td3_cfg(64), replay, seed=2)
    td3.load(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
    for k in range(1, 5):
        td3.update(k)
    torch.cuda.synchronize()
    kept = [t.clone() for t in (td3.actor_bf16, td3.actor_t_bf16, td3.critic_bf16, td3.critic_t_bf16)]
    td3.refresh()
    torch.cuda.synchronize()
    for name, a, b in zip(("actor", "actor_t"), kept[:2], (td3.actor_bf16, td3.actor_t_bf16)):
        assert torch.equal(a, b), name
    # critics: every element the updates maintain (all but the transposed blocks nothing reads:
    # the targets' W1T / W2T, the online W1T rows outside the action columns)
    for name, a, b, tgt in (("critic", kept[2], td3.critic_bf16, False), ("critic_t", kept[3], td3.critic_t_bf16, True)):
        m = td3.bf16_maintained(tgt)
        a16, b16 = a.view(torch.int16)[:m.numel()], b.view(torch.int16)[:m.numel()]
        assert torch.equal(a16[m], b16[m]), name
        assert int((~m).sum()) < m.numel() // 2, name


def test_td3_graph_replay_matches_eager():
    import torch
    import paper_2502_17496_b200 as pk
    shape, cs_, B = sg.preset("cfg1")
    replay = pk.replay_fill(20000, 17, 6, seed=3)
    outs = []
    for mode in ("eager", "graph"):
        rng = np.random.default_rng(8)
        actor = sg.actor_params(shape, rng)
        cs = sg.CriticShape(23, precision="bf16")
        c1, c2 = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
        td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(23), pk.td3_cfg(B), replay, seed=11)
        td3.load(actor, c1, c2)
        if mode == "graph":
            snap = [t.clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.critic_t)]
            td3.capture()          # capture enqueues nothing; restore state to be safe
            for t, sn in zip((td3.actor, td3.critic, td3.actor_t, td3.critic_t), snap):
                t.copy_(sn)
            td3.refresh()
            for t in (td3.m_actor, td3.v_actor, td3.m_critic, td3.v_critic, td3.adam_steps, td3.rng_counter):
                t.zero_()
            for k in range(1, 7):
                td3.replay_graph(k)
        else:
            for k in range(1, 7):
                td3.update(k)
        torch.cuda.synchronize()
        outs.append([t.cpu().clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.losses, td3.rng_counter)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_device_replay_and_rng():
    import torch
    import paper_2502_17496_b200 as pk
    n = 200_000
    r = pk.replay_fill(n, 17, 6, seed=5)
    s = r.s.cpu().numpy()
    assert abs(s.mean()) < 0.01 and abs(s.std() - 1) < 0.01 and s.max() <= 5 and s.min() >= -5
    a = r.a.cpu().numpy()
    assert a.min() >= -1 and a.max() <= 1 and abs(a.mean()) < 0.01
    d = r.d.cpu().numpy()
    assert set(np.unique(d)) <= {0.0, 1.0} and abs(d.mean() - 0.01) < 0.002
    r2 = pk.replay_fill(n, 17, 6, seed=5, rank=1)
    assert not torch.equal(r.s, r2.s)


@pytest.mark.parametrize("preset,B,T", [("cfg1", 256, 5), ("cfg3s", 100, 16), ("cfg0", 37, 7)])
def test_staged_output_scan_matches_direct_subprocess(preset, B, T, tmp_path):
    """The TMA-staged output-layer reverse scan (default) and the direct-load kernel
    (SPIKERL_OUTSCAN_DIRECT=1, a subprocess) produce bit-identical actor gradients: same per-element
    arithmetic, only the staging of the spike / mask words and the action gradients differs."""
    import os, subprocess, sys
    shape, _, _ = sg.preset(preset)
    shape = sg.with_(shape, T=T)
    p, s, g = _inputs(shape, B)
    here = run_gpu_actor(shape, B, p, s, g)
    code = (
        "import numpy as np, pickle, synthgen as sg\n"
        "from tests._parity import run_gpu_actor\n"
        f"shape, _, _ = sg.preset({preset!r}); shape = sg.with_(shape, T={T})\n"
        f"d = pickle.load(open({str(tmp_path / 'in.pkl')!r}, 'rb'))\n"
        f"out = run_gpu_actor(shape, {B}, d['p'], d['s'], d['g'])\n"
        f"pickle.dump(out['grads'], open({str(tmp_path / 'out.pkl')!r}, 'wb'))\n"
        "print('direct ok')\n")
    import pickle
    pickle.dump(dict(p=p, s=s, g=g), open(tmp_path / "in.pkl", "wb"))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, SPIKERL_OUTSCAN_DIRECT="1", PYTHONPATH=root))
    assert r.returncode == 0 and "direct ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    other = pickle.load(open(tmp_path / "out.pkl", "rb"))
    for k in here["grads"]:
        assert np.array_equal(here["grads"][k], other[k]), k


def test_nccl_single_rank_comm():
    """The NCCL path on one GPU (a world-size-1 communicator): the mean allreduce and the broadcast
    leave their buffers bit-identical, and TD3 updates with the communicator (eager and replayed
    from a captured graph, NCCL calls inside the capture) equal the updates without it bitwise."""
    import torch
    import paper_2502_17496_b200 as pk
    comm = pk.Comm(0, 1)
    x = torch.randn(1 << 20, device="cuda")
    y = x.clone()
    comm.allreduce_mean(y)
    comm.broadcast(y, 0)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    shape, _, B = sg.preset("cfg1")
    replay = pk.replay_fill(20000, 17, 6, seed=3)
    outs = []
    for use_comm, mode in ((False, "eager"), (True, "eager"), (True, "graph"), (True, "pair")):
        rng = np.random.default_rng(8)
        actor = sg.actor_params(shape, rng)
        cs = sg.CriticShape(23, precision="bf16")
        c1, c2 = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
        td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(23), pk.td3_cfg(B), replay, seed=11,
                     comm=comm if use_comm else None)
        td3.load(actor, c1, c2)
        if mode == "graph":
            snap = [t.clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.critic_t)]
            td3.capture()
            for t, sn in zip((td3.actor, td3.critic, td3.actor_t, td3.critic_t), snap):
                t.copy_(sn)
            td3.refresh()
            for t in (td3.m_actor, td3.v_actor, td3.m_critic, td3.v_critic, td3.adam_steps, td3.rng_counter):
                t.zero_()
            for k in range(1, 5):
                td3.replay_graph(k)
        elif mode == "pair":
            td3.update_pair(1)
            td3.update_pair(3)
        else:
            for k in range(1, 5):
                td3.update(k)
        torch.cuda.synchronize()
        outs.append([t.cpu().clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.losses)])
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)
    comm.close()


@pytest.mark.parametrize("preset,B", [("cfg1", 256), ("cfg3L", 8192)])
def test_actor_backward_dp_buckets_world1(preset, B):
    """The bucketed gradient mean (spikerl_actor_backward_dp: W3|Wd|bd, W2, mu|sigma|W1 allreduced on
    the comm stream as each is produced) through a one-rank NCCL communicator, eager and captured in
    a CUDA graph: bitwise the plain backward's gradient (ncclAvg over one rank is the identity), in
    the side-stream schedule (T B <= 32768) and the one-stream schedule."""
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, _ = sg.preset(preset)
    p, s, g = _inputs(shape, B, seed=31)
    comm = pk.Comm(0, 1)
    actor = pk.SpikingActor(pk.actor_cfg_from(shape), B)
    actor.load(p)
    b = actor.grad_buckets()
    assert b[0] == 0 and b[-1] == actor.n_params and b == sorted(b)
    obs = torch.from_numpy(s).cuda()
    ga = torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda()
    actor.forward(obs)
    ref = actor.backward(obs, ga).clone()
    actor.grads.zero_()
    got = actor.backward(obs, ga, comm=comm).clone()
    torch.cuda.synchronize()
    assert torch.equal(ref, got)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            actor.forward(obs)
            actor.backward(obs, ga, comm=comm)
    torch.cuda.current_stream().wait_stream(st)
    actor.grads.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(ref, actor.grads)
    comm.close()


def test_fused_allreduce_adam_world1():
    """SURVEY 8(f) NEXT #1 at world 1 (the only size this build's GPU allocation allows): the fused
    gradient-mean + Adam kernel over NCCL symmetric memory (spikerl_fused_allreduce_adam) leaves
    parameters, moments, step counts and the bf16 working copies bitwise equal to the NCCL allreduce +
    Adam launches, over four TD3 updates (single and pair form, critic and actor plans); and the
    stand-alone call equals spikerl_adam (with the sigma clamp range) bitwise."""
    import torch
    import paper_2502_17496_b200 as pk
    comm = pk.Comm(0, 1)
    try:
        g0 = comm.alloc(8)
        comm.fused_adam(g0, comm.alloc(8))
    except pk.SpikeRLError as e:
        pytest.skip(f"NCCL symmetric memory / device API unavailable here: {e}")
    n = 100_003
    rng = np.random.default_rng(3)
    g = comm.alloc(n)
    p = comm.alloc(n)
    p.copy_(torch.from_numpy(rng.standard_normal(n).astype(np.float32)))
    plan = comm.fused_adam(g, p)
    p_ref = p.clone()
    m1, v1, m2, v2 = (torch.zeros(n, device="cuda") for _ in range(4))
    c1, c2 = (torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(2))
    lib = pk.lib()
    for t in range(3):
        g.copy_(torch.from_numpy(rng.standard_normal(n).astype(np.float32)))
        pk.adam(p_ref, g, m1, v1, c1, 1e-3, clamp=(10, 200, 1e-3))
        pk._lib.check(lib.spikerl_fused_allreduce_adam(plan, pk.api._p(m2), pk.api._p(v2), pk.api._p(c2), 1e-3, 0.9,
                                                        0.999, 1e-8, 10, 200, 1e-3, pk.api._stream()), "fused")
    torch.cuda.synchronize()
    for a, b in ((p_ref, p), (m1, m2), (v1, v2), (c1, c2)):
        assert torch.equal(a, b)
    shape, _, B = sg.preset("cfg1")
    replay = pk.replay_fill(20000, 17, 6, seed=3)
    outs = []
    for fused, pair in ((False, False), (True, False), (True, True)):
        rng = np.random.default_rng(8)
        actor = sg.actor_params(shape, rng)
        cs = sg.CriticShape(23, precision="bf16")
        c1p, c2p = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
        td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(23), pk.td3_cfg(B), replay, seed=11, comm=comm,
                     fused=fused)
        td3.load(actor, c1p, c2p)
        if pair:
            td3.update_pair(1); td3.update_pair(3)
        else:
            for k in range(1, 5):
                td3.update(k)
        torch.cuda.synchronize()
        outs.append([t.cpu().clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.critic_t, td3.m_actor,
                                                td3.v_critic, td3.adam_steps, td3.actor_bf16, td3.critic_bf16)])
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)


@pytest.mark.parametrize("preset", ["cfg1", "cfg3L"])
def test_td3_pair_matches_sequential(preset):
    """spikerl_td3_update_pair(k) (update k + 1's target path and pi(s) overlapping update k) leaves
    bitwise the same state as update(k); update(k + 1): with injected minibatches / noise, with the
    device Philox draws (counter advanced by two), and replayed from a captured graph."""
    import torch
    import paper_2502_17496_b200 as pk
    shape, cs_, B = sg.preset(preset)
    replay = pk.replay_fill(20000, shape.obs_dim, shape.act_dim, seed=3)
    g = torch.Generator(device="cuda").manual_seed(5)
    idx = torch.randint(0, 20000, (2, B), device="cuda", generator=g, dtype=torch.int64)
    nz = torch.randn(2, B, shape.act_dim, device="cuda", generator=g)
    outs = {}
    for mode in ("seq", "pair", "seq_rng", "pair_rng", "pair_graph"):
        rng = np.random.default_rng(8)
        actor = sg.actor_params(shape, rng)
        cs = sg.CriticShape(cs_.in_dim, precision="bf16")
        c1, c2 = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
        td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(cs_.in_dim), pk.td3_cfg(B), replay, seed=11)
        td3.load(actor, c1, c2)
        for j in range(2):          # steps 1..4
            k = 2 * j + 1
            if mode == "seq":
                td3.update(k, idx[0], nz[0]); td3.update(k + 1, idx[1], nz[1])
            elif mode == "pair":
                td3.update_pair(k, idx, nz)
            elif mode == "seq_rng":
                td3.update(k); td3.update(k + 1)
            elif mode == "pair_rng":
                td3.update_pair(k)
            else:
                if j == 0:
                    snap = [t.clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.critic_t)]
                    td3.capture_pair()
                    for t, sn in zip((td3.actor, td3.critic, td3.actor_t, td3.critic_t), snap):
                        t.copy_(sn)
                    td3.refresh()
                    for t in (td3.m_actor, td3.v_actor, td3.m_critic, td3.v_critic, td3.adam_steps,
                              td3.rng_counter):
                        t.zero_()
                td3.replay_pair()
        torch.cuda.synchronize()
        outs[mode] = [t.cpu().clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.critic_t, td3.losses,
                                                 td3.m_actor, td3.v_critic, td3.rng_counter)]
    for a, b in zip(outs["seq"], outs["pair"]):
        assert torch.equal(a, b)
    for other in ("pair_rng", "pair_graph"):
        for a, b in zip(outs["seq_rng"], outs[other]):
            assert torch.equal(a, b), other


def _amp_td3(pk, shape, B, replay, loss_scale, interval=2000):
    rng = np.random.default_rng(8)
    actor = sg.actor_params(shape, rng)
    cs = sg.CriticShape(shape.obs_dim + shape.act_dim, precision="bf16")
    c1, c2 = sg.critic_params(cs, rng), sg.critic_params(cs, rng)
    td3 = pk.TD3(pk.actor_cfg_from(shape), pk.critic_cfg(cs.in_dim), pk.td3_cfg(B, amp_interval=interval), replay,
                 seed=11, loss_scale=loss_scale)
    td3.load(actor, c1, c2)
    return td3


def test_td3_loss_scaling_matches_unscaled():
    """Dynamic loss scaling with a power-of-two scale and no overflow changes
    nothing: dQ * 2^16 flows through bf16 roundings and fp32 sums exactly scaled, the Adam kernel
    unscales exactly; four updates (single and pair form) leave the same parameters as without it,
    and the scaler counts its finite steps (oracle state machine)."""
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, B = sg.preset("cfg1")
    replay = pk.replay_fill(20000, 17, 6, seed=3)
    g = torch.Generator(device="cuda").manual_seed(5)
    idx = torch.randint(0, 20000, (4, B), device="cuda", generator=g, dtype=torch.int64)
    nz = torch.randn(4, B, 6, device="cuda", generator=g)
    outs = []
    for scale, pair in ((None, False), (65536.0, False), (65536.0, True)):
        td3 = _amp_td3(pk, shape, B, replay, scale)
        if pair:
            td3.update_pair(1, idx[:2], nz[:2]); td3.update_pair(3, idx[2:], nz[2:])
        else:
            for k in range(1, 5):
                td3.update(k, idx[k - 1], nz[k - 1])
        torch.cuda.synchronize()
        outs.append([t.cpu().clone() for t in (td3.actor, td3.critic, td3.actor_t, td3.critic_t, td3.losses)])
        if scale is not None:
            st_c, st_a = (scale, 0), (scale, 0)
            for k in range(1, 5):
                st_c, _ = oracle.amp_step(st_c, True)
                if k % 2 == 0:
                    st_a, _ = oracle.amp_step(st_a, True)
            amp = td3.amp.cpu().numpy()
            assert (amp[0], amp[1], amp[2]) == (st_c[0], st_c[1], 0.0)
            assert (amp[4], amp[5], amp[6]) == (st_a[0], st_a[1], 0.0)
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)


def test_td3_loss_scaling_overflow_skips_and_backs_off():
    """A non-finite critic gradient (an infinite reward in the minibatch) skips the critic's Adam
    step (parameters, moments and its step count unchanged) and halves the critic's scale; the
    following finite updates proceed and the scale grows back after amp_interval finite steps."""
    import torch
    import paper_2502_17496_b200 as pk
    shape, _, B = sg.preset("cfg1")
    replay = pk.replay_fill(20000, 17, 6, seed=3)
    replay.r[:B] = float("inf")
    td3 = _amp_td3(pk, shape, B, replay, 1024.0, interval=2)
    bad = torch.arange(B, device="cuda", dtype=torch.int64)
    good = torch.arange(B, 2 * B, device="cuda", dtype=torch.int64)
    c0, m0 = td3.critic.clone(), td3.m_critic.clone()
    td3.update(1, bad)
    torch.cuda.synchronize()
    assert torch.equal(td3.critic, c0) and torch.equal(td3.m_critic, m0)
    assert int(td3.adam_steps[0]) == 0
    assert td3.amp[0].item() == 512.0 and td3.amp[1].item() == 0.0 and td3.amp[2].item() == 0.0
    td3.update(2, good)     # critic + actor: finite
    torch.cuda.synchronize()
    assert not torch.equal(td3.critic, c0) and int(td3.adam_steps[0]) == 1 and int(td3.adam_steps[2]) == 1
    assert td3.amp[0].item() == 512.0 and td3.amp[1].item() == 1.0
    assert td3.amp[4].item() == 1024.0 and td3.amp[5].item() == 1.0
    td3.update(3, good)     # second finite critic step in a row: grow
    torch.cuda.synchronize()
    assert td3.amp[0].item() == 1024.0 and td3.amp[1].item() == 0.0
    assert all(torch.isfinite(t).all() for t in (td3.critic, td3.actor, td3.m_critic, td3.v_critic))


# ------------------------------------------------------------------ fp16 actor (PAPER.md:164 FP16 AMP)
@pytest.mark.parametrize("name,B", [("cfg1", 256), ("cfg3L", 1024), ("cfg3L", 4096), ("cfg4", 64)])
def test_actor_fp16(name, B):
    """FP16 operands on the tcgen05 engine: the oracle rounds the same GEMM operands (R20 points)
    to binary16 instead of bf16; same tolerances as bf16 (actions 2e-2, gradients 1e-2 rel. L2)."""
    shape = sg.with_(sg.preset(name)[0], precision="fp16")
    p, s, g = _inputs(shape, B, seed=4)
    st = check_actor(run_gpu_actor(shape, B, p, s, g, engine="tcgen05"), shape, p, s, g)
    print(name, B, st)


@pytest.mark.parametrize("T,B", [(5, 33), (16, 19)])
def test_actor_fp16_edges(T, B):
    shape = sg.ActorShape(5, 3, pop_enc=7, pop_dec=9, n1=45, n2=161, T=T, precision="fp16")
    p, s, g = _inputs(shape, B, seed=20 + T)
    check_actor(run_gpu_actor(shape, B, p, s, g, engine="tcgen05"), shape, p, s, g)


def test_td3_fp16_actor_with_loss_scaling():
    """TD3 with the fp16 actor (bf16 critic) and dynamic loss scaling: updates run in both the
    single and the pair form with the same result, everything stays finite, the scalers count
    their finite steps, and the FP16 engine rules are enforced (no SIMT engine)."""
    import torch
    import paper_2502_17496_b200 as pk
    shape = sg.with_(sg.preset("cfg1")[0], precision="fp16")
    B = 256
    replay = pk.replay_fill(20000, 17, 6, seed=3)
    outs = []
    for pair in (False, True):
        td3 = _amp_td3(pk, shape, B, replay, 65536.0)
        if pair:
            td3.update_pair(1); td3.update_pair(3)
        else:
            for k in range(1, 5):
                td3.update(k)
        torch.cuda.synchronize()
        assert all(torch.isfinite(t).all() for t in (td3.actor, td3.critic, td3.actor_t, td3.losses))
        assert td3.amp[1].item() == 4.0 and td3.amp[5].item() == 2.0
        outs.append([t.cpu().clone() for t in (td3.actor, td3.critic, td3.actor_t)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    with pytest.raises(pk.SpikeRLError):
        pk.SpikingActor(pk.actor_cfg_from(shape, engine="simt"), 8)


# ------------------------------------------------------------------------------ bench contract
@pytest.mark.parametrize("args", [["--workload", "cfg1", "--steps", "4", "--warmup", "3"],
                                  ["--workload", "cfg0", "--steps", "4", "--warmup", "3"],
                                  ["--impl", "reference", "--workload", "cfg1", "--steps", "1", "--warmup", "1"]])
def test_bench_contract(args):
    """bench.py prints one JSON line with the contract's keys (short runs; the driver's full runs use
    the same code): value / metric / unit / timing keys, clocks, the launch count, e2e with the copied
    bytes, the live roofline with its peak and traffic, the oracle baseline; the reference arm its own
    line with impl = reference."""
    import json, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", *args, "--no-cpu-baseline"] if "--impl" not in args else
                       [sys.executable, "bench.py", *args], cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1
    assert d["e2e"]["value"] > 0 and "unit" in d["e2e"]
    if "--impl" in args:
        assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
        assert d["e2e"]["h2d_bytes_per_step"] == 0
        return
    assert d["config"]["workload"].startswith(args[1])
    assert d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    roof = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "timing"):
        assert k in roof, k
    assert 0 < roof["frac"] <= 1.5 and roof["peak"] > 0
