"""World-size-2 `gloo` tests of the data-parallel host logic (CPU, no GPU needed).

Only one GPU is available to this build, so the N > 1 path is covered here: the NCCL-id
rendezvous the library uses (PAPER.md:135 broadcast_weights runs over the resulting comm), and
the DP semantics of the update — per-rank shards, gradient mean over ranks (PAPER.md:135
average_gradients; PAPER.md:144 DDP), replicas staying bitwise identical, and W ranks x B
matching 1 rank x W*B.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_id(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    import ctypes as C
    from paper_2502_17496_b200 import _lib
    buf = (C.c_ubyte * 128)()
    ok = True
    if rank == 0:
        st = _lib.lib().spikerl_comm_get_unique_id(buf)
        ok = st == 0
    obj = [bytes(buf) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    q.put((rank, ok, obj[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_unique_id_rendezvous_over_gloo():
    from paper_2502_17496_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    try:
        C = __import__("ctypes")
        b = (C.c_ubyte * 128)()
        if _lib.lib().spikerl_comm_get_unique_id(b) != 0:
            pytest.skip("NCCL unique id unavailable in this container: " + _lib.last_error())
    except OSError as e:
        pytest.skip(str(e))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_id, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert res[0][2] == res[1][2] and len(res[0][2]) == 128 and any(res[0][2])


def _worker_td3(rank, world, port, q, n_steps, scheme="A"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    import oracle
    import synthgen as sg

    def allreduce_mean(dicts):
        out = []
        for d in dicts:
            o = {}
            for k, v in d.items():
                t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
                if scheme == "B":      # DDP: gradients pre-divided by the world size, then summed
                    t = t / world
                    dist.all_reduce(t)
                    o[k] = t.numpy()
                else:                  # MPI average_gradients: sum over ranks, then divide
                    dist.all_reduce(t)
                    o[k] = (t / world).numpy()
            out.append(o)
        return out

    shape = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5, precision="fp32")
    cs = sg.CriticShape(5, 16, 16, precision="fp32")
    hp = sg.TD3Hyper()
    # scheme A: each rank draws its own init and rank 0's is broadcast (PAPER.md:135
    # broadcast_weights); scheme B: every rank builds the same seeded init (DDP's start state)
    rng = np.random.default_rng(0 if scheme == "B" else 77 * rank)
    st = oracle.init_state(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
    if scheme == "A":
        rng0 = np.random.default_rng(0)
        ref = oracle.init_state(sg.actor_params(shape, rng0), sg.critic_params(cs, rng0), sg.critic_params(cs, rng0))

        def bcast(a):
            t = torch.from_numpy(np.ascontiguousarray(a) if rank == 0 else np.zeros_like(a))
            dist.broadcast(t, 0)
            return t.numpy()

        def walk(x):
            if isinstance(x, dict):
                return {k: walk(v) for k, v in x.items()}
            if isinstance(x, (list, tuple)):
                return type(x)(walk(v) for v in x)
            if isinstance(x, np.ndarray):
                return bcast(x)
            return x
        st = walk(st)
        assert all(np.array_equal(st["actor"][k], ref["actor"][k]) for k in ref["actor"])
    B = 6
    for k in range(1, n_steps + 1):
        brng = np.random.default_rng(1000 + k)  # the global batch of step k, split by rank
        full = sg.replay_batch(brng, B * world, 3, 2)
        eps = sg.target_noise(brng, B * world, 2)
        sl = slice(rank * B, (rank + 1) * B)
        shard = {kk: v[sl] for kk, v in full.items()}
        st, info = oracle.td3_update(st, shape, cs, hp, shard, eps[sl], k, allreduce=allreduce_mean)
    flat = np.concatenate([np.ravel(st["actor"][kk]) for kk in sorted(st["actor"])] +
                          [np.ravel(c[kk]) for c in st["c"] for kk in sorted(c)])
    q.put((rank, flat))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_td3_equivalence():
    """2 ranks x B == 1 rank x 2B (mean losses), and both replicas stay identical."""
    import oracle
    import synthgen as sg
    n_steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_td3, args=(r, 2, port, q, n_steps)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert np.array_equal(res[0], res[1])                       # replicas bitwise identical
    # single process on the concatenated batch
    shape = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5, precision="fp32")
    cs = sg.CriticShape(5, 16, 16, precision="fp32")
    hp = sg.TD3Hyper()
    rng = np.random.default_rng(0)
    st = oracle.init_state(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
    for k in range(1, n_steps + 1):
        brng = np.random.default_rng(1000 + k)
        full = sg.replay_batch(brng, 12, 3, 2)
        eps = sg.target_noise(brng, 12, 2)
        st, _ = oracle.td3_update(st, shape, cs, hp, full, eps, k)
    flat = np.concatenate([np.ravel(st["actor"][kk]) for kk in sorted(st["actor"])] +
                          [np.ravel(c[kk]) for c in st["c"] for kk in sorted(c)])
    assert np.allclose(res[0], flat, rtol=1e-5, atol=1e-9)


def test_scheme_a_equals_scheme_b():
    """PAPER.md:135 (MPI: broadcast_weights + average_gradients) and PAPER.md:144 (DDP: same init,
    gradients pre-divided then summed) give bit-identical replicas at world size 2: division by 2
    is exact, so sum-then-divide and divide-then-sum round identically."""
    ctx = mp.get_context("spawn")
    out = {}
    for scheme in ("A", "B"):
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_worker_td3, args=(r, 2, port, q, 3, scheme)) for r in range(2)]
        for p in ps:
            p.start()
        res = dict(q.get(timeout=300) for _ in range(2))
        for p in ps:
            p.join(timeout=60)
        assert np.array_equal(res[0], res[1])
        out[scheme] = res[0]
    assert np.array_equal(out["A"], out["B"])


def _worker_buckets(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    import ctypes as C
    import oracle
    import synthgen as sg
    from paper_2502_17496_b200 import _lib, actor_cfg_from, pack_actor
    shape = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5, precision="fp32")
    cfg = actor_cfg_from(shape)
    bounds = (C.c_size_t * 4)()
    assert _lib.lib().spikerl_actor_grad_buckets(C.byref(cfg), bounds) == 0
    rng = np.random.default_rng(0)
    p = sg.randomize_actor(shape, rng)
    s = sg.observations(rng, 8, 3)
    g = sg.action_grads(rng, 8, 2)
    sl = slice(4 * rank, 4 * rank + 4)
    _, tape = oracle.actor_forward(p, shape, s[sl])
    grad = oracle.actor_backward(p, shape, tape, g[sl])
    flat = pack_actor(cfg, {k: v.astype(np.float32) for k, v in grad.items()}, device="cpu").double()
    whole = flat.clone()
    dist.all_reduce(whole)
    whole /= world
    bucketed = flat.clone()
    for i in (2, 1, 0):            # the library's completion order: W3|Wd|bd, W2, mu|sigma|W1
        seg = bucketed[bounds[i]:bounds[i + 1]]
        dist.all_reduce(seg)
        seg /= world
    q.put((rank, list(bounds), whole.numpy(), bucketed.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_bucketed_allreduce_matches_whole():
    """The library's gradient buckets (spikerl_actor_grad_buckets: host logic) tile the flat actor
    gradient in order, and a mean allreduced bucket by bucket in the library's completion order equals
    the whole-vector mean bitwise on both ranks, which equals the fp32-packed oracle gradient of the
    concatenated batch over 2 (PAPER.md:135 average_gradients)."""
    import oracle
    import synthgen as sg
    from paper_2502_17496_b200 import actor_cfg_from, pack_actor, _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_buckets, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in ps:
        p.join(timeout=60)
    bounds = res[0][0]
    shape = sg.ActorShape(3, 2, pop_enc=5, pop_dec=4, n1=12, n2=10, T=5, precision="fp32")
    cfg = actor_cfg_from(shape)
    n = pack_actor(cfg, sg.actor_params(shape, np.random.default_rng(0)), device="cpu").numel()
    assert bounds[0] == 0 and bounds[-1] == n and all(a < b for a, b in zip(bounds, bounds[1:]))
    for r in (0, 1):
        assert np.array_equal(res[r][1], res[r][2])
    assert np.array_equal(res[0][2], res[1][2])
    rng = np.random.default_rng(0)
    p = sg.randomize_actor(shape, rng)
    s = sg.observations(rng, 8, 3)
    g = sg.action_grads(rng, 8, 2)
    _, tape = oracle.actor_forward(p, shape, s)
    full = oracle.actor_backward(p, shape, tape, g)
    ref = pack_actor(cfg, {k: (v / 2).astype(np.float32) for k, v in full.items()}, device="cpu").double().numpy()
    assert np.allclose(res[0][2], ref, rtol=1e-6, atol=1e-7)


def test_bench_sharding_arithmetic():
    """bench.py's per-rank split of configs[4] and weak-scaling accounting."""
    import bench
    import synthgen as sg
    _, _, Bg = sg.preset("cfg4")
    for world in (1, 2, 4, 8):
        assert (Bg // world) * world == Bg
    assert bench.METRIC.startswith("TD3 spiking-actor updates/sec")
