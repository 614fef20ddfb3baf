#!/usr/bin/env python
"""Benchmark of the SpikeRL hot path on B200 (contract: see DESIGN.md "Measurement").

  python bench.py [--gpus N --steps K --warmup W] [--workload cfg0|cfg1|cfg2|cfg3s|cfg3L|cfg4]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (data parallel)
  python bench.py --impl reference      (the CPU oracle, timed on the host cores)

One JSON line on rank 0. The default workload is configs[4] (BASELINE.json's large-batch
config, the largest that fits one GPU): a step is one actor forward + surrogate-gradient BPTT +
gradient allreduce over the rank's shard of the 65 536-row global batch (strong scaling). The same
line carries, under "td3", configs[3] at per-rank batch 4096 (the TD3 throughput regime, weak
scaling): a step there is one TD3 update (replay sample -> target actor -> target critics -> critic
fwd/bwd -> allreduce -> Adam -> [delayed actor fwd/BPTT, allreduce, Adam, Polyak]). Inputs are
device-resident when the timed region starts; `e2e` re-times the same step through the public
API with its inputs copied from pinned host memory and its result read back every step. The
roofline kernel is timed live inside the timed region (event pairs around its launches on its own
stream, recorded as graph event nodes).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# diagnostics: SPIKERL_BENCH_COMM=1 runs the N > 1 code path (NCCL communicator, allreduce inside the
# captured graph) on a single GPU with a world-size-1 communicator
FORCE_COMM = os.environ.get("SPIKERL_BENCH_COMM", "0") == "1"
METRIC = "TD3 spiking-actor updates/sec at 1/2/4/8 B200; actor fwd+bwd samples/sec"
SIMT_FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # guide: 148 SMs x 128 FP32 lanes x FMA x max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg0", "cfg1", "cfg2", "cfg3s", "cfg3L", "cfg4"])
    ap.add_argument("--no-td3-extra", action="store_true", help="cfg4: skip the configs[3] B=4096 TD3 keys")
    ap.add_argument("--eager", action="store_true", help="actor workloads: eager launches instead of a graph")
    ap.add_argument("--fused-dp", action="store_true",
                    help="TD3 with a communicator: the fused gradient-mean + Adam kernel over NCCL symmetric memory")
    ap.add_argument("--single-graphs", action="store_true",
                    help="TD3: replay one graph per update instead of overlapped update pairs")
    ap.add_argument("--engine", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replay-size", type=int, default=1_000_000)
    return ap.parse_args()


def peaks():
    p = {"hbm_gbs": 6546.6, "bf16_tflops": 1631.2, "bf16_tflops_sustained": 1376.6, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["src"] = "measured"
    except Exception:
        pass
    return p


# ---------------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons during the timed region: NVML polled every ~2 ms from a thread
    (a latency-bound timed region lasts only tens of ms), nvidia-smi as the fallback."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nvml = None

    def start(self):
        if self.nvml is not None:
            self.samples, self.reasons, self.stop_flag = [], 0, False
            nv = self.nvml

            def poll():
                while not self.stop_flag:
                    try:
                        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                        self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        self._start_smi()

    def _stop_nvml(self):
        self.stop_flag = True
        self.t.join(timeout=2)
        nv = self.nvml
        mx = None
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            pass
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
        reasons = sorted(n for bit, n in names.items() if self.reasons & bit)
        sm = sorted(self.samples)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(sm), "source": "nvml"}

    def _start_smi(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _energy_mj(self):
        try:
            return self.nvml.nvmlDeviceGetTotalEnergyConsumption(self.h) if self.nvml is not None else None
        except Exception:
            return None

    def stop(self):
        if self.nvml is not None:
            return self._stop_nvml()
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0])); mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------- dist
def dist_init(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x, world):
    import torch
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------------- workloads
def build_td3(name, world, rank, engine, replay_size, seed=0, fused=False):
    import numpy as np
    import synthgen as sg
    import paper_2502_17496_b200 as pk
    shape, cshape, B = sg.preset(name)
    acfg = pk.actor_cfg_from(shape, engine=engine)
    ccfg = pk.critic_cfg(cshape.in_dim, precision=shape.precision)
    replay = pk.replay_fill(replay_size, shape.obs_dim, shape.act_dim, seed=seed, rank=rank)
    comm = pk.Comm(rank, world) if (world > 1 or FORCE_COMM) else None
    td3 = pk.TD3(acfg, ccfg, pk.td3_cfg(B), replay, seed=seed, comm=comm, fused=fused)
    rng = np.random.default_rng(seed)
    td3.load(sg.actor_params(shape, rng), sg.critic_params(cshape, rng), sg.critic_params(cshape, rng))
    return td3, shape, B


def l2_flush(buf):
    """Evict L2 by READING a buffer twice its size (clean lines: a write flush would leave ~126 MB of
    dirty lines whose write-back the next timed kernel pays for)."""
    import torch
    torch.sum(buf)


def energy_window(run_step, sampler, seconds=1.5):
    """GPU energy per step (NVML total-energy counter, mJ; it updates too coarsely for the short timed
    region): steps run back to back for >= `seconds` after the timed region, energy difference over
    that window / steps. PAPER.md §IV-B GPS-UP context (B200 side only)."""
    import torch
    torch.cuda.synchronize()
    e0 = sampler._energy_mj()
    if e0 is None:
        return None
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds or n < 3:
        run_step(n)
        n += 1
        if n % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    dt, e1 = time.time() - t0, sampler._energy_mj()
    j = (e1 - e0) / 1e3
    return {"joules": round(j, 3), "steps": n, "seconds": round(dt, 3), "avg_watts": round(j / dt, 1),
            "source": "nvml total energy counter, steps back to back after the timed region"}


def time_steps(run_step, K, flush_buf, world, after_step=None):
    """Per-step CUDA events on the launching stream; L2 flushed between steps (outside events).
    after_step (optional) runs after each step's end event, outside the timed interval (the live
    kernel watch synchronises there and reads its event pairs)."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    barrier(world)
    for k in range(K):
        if flush_buf is not None:
            l2_flush(flush_buf)
        evs[k][0].record()
        run_step(k)
        evs[k][1].record()
        if after_step is not None:
            after_step(k)
    torch.cuda.synchronize()
    barrier(world)
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    return max_over_ranks(total_ms, world)


def dominant_kernel(summary, pk_peaks, live, timed_ms, workload, clocks=None, long_step=False):
    """The largest kernel of the step (by the profiling pass's launch list) against its roofline.
    `live` = (launches, total_ms) of that kernel measured inside the timed region (Watch); the
    algorithmic work per launch is the launcher's attribution (flops or bytes). Tensor-bound
    kernels are judged against the burst bf16 peak (cuBLAS 8192^3 at full clock), the stricter of
    the two measured figures; for a long step whose sampled clock sagged below 95% of max the
    sustained figure and the frac against it are reported beside as context."""
    best = max(summary, key=lambda e: e["total_ms"])
    n_live, ms_live = live
    avg_s = ms_live / n_live / 1e3
    extra = {}
    if best["bound"] == "tensor":
        per = best["flops"] / best["launches"]
        sagged = bool(clocks and clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
                      and clocks["sm_mhz"] < 0.95 * clocks["sm_max_mhz"])
        peak = pk_peaks["bf16_tflops"]
        if long_step and sagged and pk_peaks.get("bf16_tflops_sustained"):
            ps = pk_peaks["bf16_tflops_sustained"]
            extra = {"peak_sustained": ps, "frac_vs_sustained": round(per / avg_s / 1e12 / ps, 5)}
        ach, unit, bound = per / avg_s / 1e12, "TFLOP/s", "tensor"
    elif best["bound"] == "alu":
        per = best["flops"] / best["launches"]
        peak = SIMT_FP32_PEAK_TFLOPS
        ach, unit, bound = per / avg_s / 1e12, "TFLOP/s", "alu"
    else:
        per = best["bytes"] / best["launches"]
        peak = pk_peaks["hbm_gbs"]
        ach, unit, bound = per / avg_s / 1e9, "GB/s", "hbm"
    # DRAM bytes per launch from one ncu --set full capture of this kernel AT THIS WORKLOAD
    # (profiles/ncu_traffic.json, keyed "<workload>:<kernel>"); null when none was captured
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{workload}:{best['name']}")
    except Exception:
        pass
    return {"kernel": best["name"], "bound": bound, "achieved": round(ach, 3), "peak": peak, "unit": unit,
            "frac": round(ach / peak, 5), "traffic": traffic, "work_per_launch": per,
            "avg_launch_us": round(avg_s * 1e6, 3), "launches_timed": n_live,
            "timing": "live: CUDA event pair around every launch of this kernel, on its launch stream, in a second "
                      "timed loop of as many steps replaying the same step graph captured with those event nodes "
                      "(the value's loop carries none); in a DAG with concurrent branches a launch's interval "
                      "includes sharing the GPU with the kernels overlapping it",
            "share_of_step": round(ms_live / max(timed_ms, 1e-12), 4),
            "peak_src": pk_peaks["src"] if bound != "alu" else "derived (guide: 148 SM x 128 lanes x 2 x 1.965 GHz)",
            "peak_kind": "burst" if bound == "tensor" else ("copy" if bound == "hbm" else "derived"), **extra}


def cpu_baseline_td3(name, seconds=12.0, min_steps=4):
    import numpy as np
    import oracle
    import synthgen as sg
    shape, cs, B = sg.preset(name)
    rng = np.random.default_rng(0)
    st = oracle.init_state(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))
    hp = sg.TD3Hyper()
    t0 = time.time()
    k = 0
    while k < min_steps or (time.time() - t0 < seconds and k % 2 == 0) or k % 2 == 1:
        k += 1
        st, _ = oracle.td3_update(st, shape, cs, hp, sg.replay_batch(rng, B, shape.obs_dim, shape.act_dim),
                                  sg.target_noise(rng, B, shape.act_dim), k)
        if time.time() - t0 > 4 * seconds:
            break
    dt = time.time() - t0
    return {"value": round(k * B / dt, 3), "unit": "samples/s", "updates_per_s": round(k / dt, 4),
            "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"{k} full TD3 updates of {name} (B={B}, half with the delayed actor step), numpy fp64 oracle"}


class HostEnergy:
    """Host CPU energy from the RAPL powercap counters (/sys/class/powercap/*/energy_uj), when the box
    exposes them; None otherwise (the r01/r02 boxes do not)."""

    def __init__(self):
        import glob
        self.files = [f for f in glob.glob("/sys/class/powercap/*/energy_uj") if os.access(f, os.R_OK)]

    def read_j(self):
        if not self.files:
            return None
        try:
            return sum(int(open(f).read()) for f in self.files) / 1e6
        except Exception:
            return None


def cpu_baseline_actor(name, B_sample=16, seconds=12.0, threads=None):
    import numpy as np
    import oracle
    import synthgen as sg
    from threadpoolctl import threadpool_limits
    shape, _, B = sg.preset(name)
    rng = np.random.default_rng(0)
    p = sg.actor_params(shape, rng)
    he = HostEnergy()
    with threadpool_limits(limits=threads):
        e0 = he.read_j()
        t0 = time.time()
        n = 0
        while n == 0 or time.time() - t0 < seconds:
            s = sg.observations(rng, B_sample, shape.obs_dim)
            a, tape = oracle.actor_forward(p, shape, s)
            oracle.actor_backward(p, shape, tape, sg.action_grads(rng, B_sample, shape.act_dim))
            n += B_sample
        dt = time.time() - t0
        e1 = he.read_j()
    out = {"value": round(n / dt, 3), "unit": "samples/s", "cores": threads or len(os.sched_getaffinity(0)),
           "kind": "oracle",
           "sample": f"{n} samples of {name} actor fwd+BPTT in batches of {B_sample} (extrapolates linearly in B)"}
    if e0 is not None and e1 is not None:
        out["host_joules_per_sample"] = round((e1 - e0) / n, 6)
    return out


def gps_up(gpu_value, energy, cpu):
    """The paper's GPS-UP view (§IV-B; R29: phi labels the baseline):
    Speedup = T_oracle / T_gpu, Powerup = P_oracle / P_gpu, Greenup = Speedup x Powerup = the energy
    per sample ratio. The GPU side is measured (NVML counter); the host side needs RAPL counters,
    which these boxes do not expose, so Powerup and Greenup stay null there. Context only."""
    out = {"speedup": round(gpu_value / cpu["value"], 1) if cpu and cpu.get("value") else None,
           "gpu_joules_per_sample": None, "host_joules_per_sample": cpu.get("host_joules_per_sample") if cpu else None,
           "powerup": None, "greenup": None}
    if energy and energy.get("samples_per_joule"):
        out["gpu_joules_per_sample"] = round(1.0 / energy["samples_per_joule"], 9)
    if out["gpu_joules_per_sample"] and out["host_joules_per_sample"]:
        out["greenup"] = round(out["host_joules_per_sample"] / out["gpu_joules_per_sample"], 1)
        out["powerup"] = round(out["greenup"] / out["speedup"], 3) if out["speedup"] else None
    else:
        out["why_null"] = "host CPU energy not observable on this box (no readable RAPL powercap counters)"
    return out


# ---------------------------------------------------------------------------------- ours
def _profile_pass(fn):
    """Eager pass with CUDA events around every library launch: which kernel dominates and the
    algorithmic work its launcher attributes to it (the timing itself is re-measured live)."""
    import torch
    from paper_2502_17496_b200 import _lib
    torch.cuda.synchronize()
    _lib.prof_enable(True)
    fn()
    torch.cuda.synchronize()
    summ = _lib.prof_summary()
    global _LAST_TIMELINE
    _LAST_TIMELINE = _lib.prof_timeline()
    _lib.prof_enable(False)
    return summ


_LAST_TIMELINE = []


def _breakdown(summ):
    return sorted([{k: (round(v, 4) if isinstance(v, float) else v) for k, v in e.items()} for e in summ],
                  key=lambda e: -e["total_ms"])[:12]


def _capture(fn):
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return g


def run_td3(args, rank, world, workload):
    import torch
    import paper_2502_17496_b200 as pk
    from paper_2502_17496_b200 import _lib
    td3, shape, B = build_td3(workload, world, rank, args.engine, args.replay_size, fused=args.fused_dp)
    # updates 2j+1, 2j+2 as one overlapped graph (spikerl_td3_update_pair: bitwise the same state as
    # two sequential updates, tested) unless --single-graphs
    pair = td3.hp.policy_delay == 2 and not args.single_graphs
    lib = pk.lib()
    launches = {}

    td3.update(1)                   # first launches (module loading, tensor maps) outside the profile
    td3.update(2)
    if pair:
        td3.update_pair(3)

    def prof_fn():
        for k in (1, 2):            # launches per phase, counted from an eager enqueue
            lib.spikerl_launch_count(1)
            td3.update(k)
            launches[k % 2] = lib.spikerl_launch_count(1)
        if pair:
            lib.spikerl_launch_count(1)
            td3.update_pair(3)
            launches["pair"] = lib.spikerl_launch_count(1)
    summ = _profile_pass(prof_fn)
    dom = max(summ, key=lambda e: e["total_ms"])["name"]
    # at most two watched launches per replayed pair: each event node in the graph cuts a programmatic
    # (PDL) edge and costs a few microseconds, which at configs[1] would itself move ms_per_step
    watch = _lib.Watch(dom, 2)
    td3.capture()
    # The watched graph (event nodes around the dominant kernel's launches) is a second capture of the
    # same pair; the value is timed on the plain one: at configs[1] the two event nodes cost ~9 us per
    # update (A/B r02), which would otherwise be charged to the method. SPIKERL_BENCH_WATCH=0: no
    # watched loop (the roofline then falls back to the eager profiling pass).
    armed = os.environ.get("SPIKERL_BENCH_WATCH", "1") != "0"
    watched_graph, per = None, 0
    if pair:
        if armed:
            watch.arm()
            td3.capture_pair()
            per = watch.used()
            _lib.Watch.off()
            watched_graph = td3.pair_graph
        td3.capture_pair()
    torch.cuda.synchronize()
    flush = None if args.no_flush else torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    step0 = [6 if pair else 2]

    def graph_step(k):
        td3.replay_graph(step0[0] + k)

    if pair:
        for k in range(max(1, args.warmup // 2)):
            td3.replay_pair()
        step0[0] += 2 * max(1, args.warmup // 2)
    else:
        for k in range(args.warmup):
            graph_step(k)
        step0[0] += args.warmup
    torch.cuda.synchronize()
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    live = None
    if pair:
        npair = args.steps // 2

        total_ms = time_steps(lambda k: td3.replay_pair(), npair, flush, world) if npair else 0.0
        step0[0] += 2 * npair
        if args.steps % 2:
            total_ms += time_steps(graph_step, 1, flush, world)
            step0[0] += 1
        gpu_launches = npair * launches["pair"] + (launches[1] if args.steps % 2 else 0)
        if watched_graph is not None and npair:
            def after(k):
                torch.cuda.synchronize()
                watch.collect(per)
            # the same number of pairs again, replaying the watched capture (same flush, same work),
            # after one untimed replay (the graph's upload)
            watched_graph.replay()
            torch.cuda.synchronize()
            time_steps(lambda k: watched_graph.replay(), npair, flush, world, after_step=after)
            step0[0] += 2 * npair + 2
            live = (watch.launches, watch.total_ms)
    else:
        total_ms = time_steps(graph_step, args.steps, flush, world)
        gpu_launches = sum(launches[(step0[0] + k) % 2] for k in range(args.steps))
        step0[0] += args.steps
    clocks = clk.stop()
    secs = total_ms / 1e3
    value = args.steps * B * world / secs
    out = {"metric": METRIC, "value": round(value, 2), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 5), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if shape.precision == "bf16" else "f32",
           "data": "synthetic (device-resident replay shard filled with Philox; configs[1] distributions)",
           "updates_per_s": round(args.steps / secs, 3),
           "config": {"workload": f"{workload}: TD3 update, spiking actor obs {shape.obs_dim} act "
                                  f"{shape.act_dim} pop 10/10 hidden {shape.n1}-{shape.n2} T={shape.T}, twin critics "
                                  f"{shape.obs_dim + shape.act_dim}->256->256->1",
                      "global_batch": B * world, "per_rank_batch": B, "replay_per_rank": args.replay_size,
                      "parallelism": f"dp{world}", "engine": args.engine,
                      "l2": ("flushed between timed pairs of updates (256 MB read, outside the events)" if pair
                             else "flushed between timed steps (256 MB read, outside the events)")
                      if flush is not None else "not flushed", "cuda_graph": True,
                      "graph": "update pairs (k odd, k + 1 overlapped)" if pair else "one graph per update",
                      "dp_optimiser": ("fused gradient mean + Adam over NCCL symmetric memory"
                                       if td3.fused_plans[0] is not None else
                                       ("bucketed NCCL allreduce + Adam" if td3.comm is not None else "none (1 GPU)"))},
           "clocks": clocks, "gpu_launches": int(gpu_launches)}
    if pair and step0[0] % 2 == 0:
        en = energy_window(lambda k: td3.replay_pair(), clk)   # each call = two updates
        if en:
            en["steps"] *= 2
    else:
        en = energy_window(lambda k: td3.replay_graph(step0[0] + k), clk)
    if en:
        step0[0] += en["steps"]
        en["joules_per_update"] = round(en["joules"] / en["steps"], 6)
        en["samples_per_joule"] = round(en["steps"] * B / max(en["joules"], 1e-9), 1)
        out["energy"] = en
    # e2e: minibatch from pinned host memory every step + loss read-back, through the public API
    if not args.no_e2e:
        out["e2e"] = e2e_td3(args, rank, world, td3, shape, B, pair=pair)
    if live is None:   # --single-graphs (diagnostic): no live watch; the eager profiling pass stands in
        d = [e for e in summ if e["name"] == dom][0]
        live = (d["launches"], d["total_ms"])
    out["roofline"] = dominant_kernel(summ, peaks(), live, total_ms, workload)
    iso = isolated_actor_kernel(td3, B, out["roofline"])
    if iso:
        out["roofline"]["isolated"] = iso
    if not pair or watched_graph is None:
        out["roofline"]["timing"] = "eager profiling pass (events around every launch); diagnostic run"
    else:
        out["roofline"]["timing"] = ("live: CUDA event pair around every launch of this kernel, on its launch stream, "
                                     "in a second timed loop of as many pairs replaying the same update-pair graph "
                                     "captured with those event nodes (the value's loop carries none: they cost "
                                     "~9 us per update at configs[1]); in a DAG with concurrent branches a launch's "
                                     "interval includes sharing the GPU with the kernels overlapping it")
    out["kernel_breakdown"] = _breakdown(summ)
    return out


def isolated_actor_kernel(td3, B, roof):
    """Context for a dominant actor kernel of a TD3 DAG, whose live interval includes sharing the GPU
    with the concurrent branches: the same kernel's mean duration when nothing else runs (an actor of
    the same shape and parameters, eager forward + backward on one stream, events around every
    launch, after one warm-up pass)."""
    import torch
    import paper_2502_17496_b200 as pk
    from paper_2502_17496_b200 import _lib
    name = roof.get("kernel", "")
    if not (name.startswith("lif_") or name.startswith("enc_")) or roof.get("bound") != "tensor":
        return None
    actor = pk.SpikingActor(td3.acfg, B)
    actor.params.copy_(td3.actor)
    actor.refresh()
    g = torch.Generator(device="cuda").manual_seed(1)
    obs = torch.clamp(torch.randn(B, td3.acfg.obs_dim, device="cuda", generator=g), -5, 5)
    ga = torch.randn(B, td3.acfg.act_dim, device="cuda", generator=g)

    def fb():
        for _ in range(3):
            actor.forward(obs)
            actor.backward(obs, ga)
    fb()
    torch.cuda.synchronize()
    _lib.prof_enable(True)
    fb()
    torch.cuda.synchronize()
    summ = _lib.prof_summary()
    _lib.prof_enable(False)
    e = [x for x in summ if x["name"] == name]
    if not e:
        return None
    avg_s = e[0]["total_ms"] / e[0]["launches"] / 1e3
    ach = roof["work_per_launch"] / avg_s / 1e12
    return {"avg_launch_us": round(avg_s * 1e6, 3), "achieved": round(ach, 3), "frac": round(ach / roof["peak"], 5),
            "how": "the same kernel alone: an actor of this shape and these parameters, eager forward + backward on "
                   "one stream, CUDA events around each launch (context; the live figure above is the DAG's)"}


def e2e_td3(args, rank, world, td3_dev, shape, B, pair=False):
    """End to end through the public API: every update's minibatch is copied from pinned host memory
    (5 H2D copies per update) and the losses are read back to pinned host memory; the timed region
    contains the copies. pair: each timed iteration is one captured graph of [H2D copies of two
    minibatches -> spikerl_td3_update_pair -> D2H of the losses] (one graph per pair of host buffers);
    otherwise an eager TD3.update per update."""
    import numpy as np
    import torch
    import paper_2502_17496_b200 as pk
    S, A = shape.obs_dim, shape.act_dim
    per = 2 * S + A + 2
    nbuf = 8
    rng = np.random.default_rng(100 + rank)
    host = [pk.replay_from_host(__import__("synthgen").replay_batch(rng, B, S, A), device="cpu") for _ in range(nbuf)]
    host = [pk.ReplayShard(*(t.pin_memory() for t in (h.s, h.a, h.r, h.s2, h.d))) for h in host]
    f32 = dict(dtype=torch.float32, device="cuda")
    nb = 2 if pair else 1
    # device staging = a replay of nb B rows whose five arrays are views of ONE buffer, so a pinned
    # host buffer with the same layout arrives in a single H2D copy. pair: two such slots (rows
    # [0, 2B) and [2B, 4B) of the staging replay, array by array), so the copy of the next pair's
    # minibatches overlaps the current pair's updates
    nslot = 2 if pair else 1
    dev = torch.empty(nslot * nb * B * per, **f32)

    def views(buf, n=None):
        n = nb * B if n is None else n
        o, out = 0, []
        for w in (S, A, 1, S, 1):
            v = buf[o:o + n * w]
            out.append(v.view(n, w) if w > 1 else v)
            o += n * w
        return pk.ReplayShard(*out)

    rs = views(dev, nslot * nb * B)
    if pair:   # pinned host buffers, one per pair of pool minibatches, in the staging layout
        packed = []
        for g_i in range(nbuf // 2):
            hb = torch.empty(nb * B * per, dtype=torch.float32).pin_memory()
            hv = views(hb)
            for j in range(2):
                h = host[2 * g_i + j]
                for src, dst in ((h.s, hv.s), (h.a, hv.a), (h.r, hv.r), (h.s2, hv.s2), (h.d, hv.d)):
                    dst[j * B:(j + 1) * B].copy_(src)
            packed.append(hb)
    td3 = pk.TD3(td3_dev.acfg, td3_dev.ccfg, td3_dev.hp, rs, seed=1, comm=td3_dev.comm)
    for t_src, t_dst in ((td3_dev.actor, td3.actor), (td3_dev.actor_t, td3.actor_t), (td3_dev.critic, td3.critic),
                         (td3_dev.critic_t, td3.critic_t)):
        t_dst.copy_(t_src)
    td3.refresh()
    idx = torch.arange(nb * B, dtype=torch.int64, device="cuda").view(nb, B)
    idx_slot = [idx + sl * nb * B for sl in range(nslot)]
    loss_host = torch.empty(2, dtype=torch.float32).pin_memory()

    def h2d(h, j):
        for src, dst in ((h.s, rs.s), (h.a, rs.a), (h.r, rs.r), (h.s2, rs.s2), (h.d, rs.d)):
            dst[j * B:(j + 1) * B].copy_(src, non_blocking=True)          # one cudaMemcpyAsync H2D each

    if pair:
        hv = [views(packed[g_i]) for g_i in range(len(packed))]

        def h2d_slot(g_i, sl):   # pair g_i's two minibatches into staging slot sl: one H2D per array
            dv = [rs.s, rs.a, rs.r, rs.s2, rs.d]
            for src, dst in zip((hv[g_i].s, hv[g_i].a, hv[g_i].r, hv[g_i].s2, hv[g_i].d), dv):
                dst[sl * nb * B:(sl + 1) * nb * B].copy_(src, non_blocking=True)

        graphs = []
        cs, cp = torch.cuda.Stream(), torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            for g_i in range(len(packed)):   # an even count: graph g_i reads slot g_i % 2
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    cp.wait_stream(cs)
                    with torch.cuda.stream(cp):   # the next pair's minibatches, during this pair's updates
                        h2d_slot((g_i + 1) % len(packed), (g_i + 1) % 2)
                    td3.update_pair(1, indices=idx_slot[g_i % 2])
                    cs.wait_stream(cp)
                    loss_host.copy_(td3.losses, non_blocking=True)
                graphs.append(g)
        torch.cuda.current_stream().wait_stream(cs)
        h2d_slot(0, 0)                       # the first pair's data (every later copy is inside a step)
        torch.cuda.synchronize()

        def step(k):
            graphs[k % len(graphs)].replay()

        nw = -(-max(1, args.warmup // 2) // len(graphs)) * len(graphs)   # whole cycles: graph 0 next
        for k in range(nw):
            step(k)
        npair = max(1, args.steps // 2)
        total_ms = time_steps(step, npair, None, world)
        torch.cuda.synchronize()
        n_upd = 2 * npair
        path = ("graphs of [H2D copies of the next two pinned host minibatches on a copy stream || "
                "spikerl_td3_update_pair on the current ones -> D2H of the losses] per two updates "
                "(TD3.update_pair through the C ABI; double-buffered staging)")
    else:
        def step(k):
            h2d(host[k % nbuf], 0)
            td3.update(k + 1, indices=idx[0])
            loss_host.copy_(td3.losses, non_blocking=True)

        for k in range(args.warmup):
            step(k)
        total_ms = time_steps(step, args.steps, None, world)
        torch.cuda.synchronize()
        n_upd = args.steps
        path = "TD3.update (eager C-ABI call) fed from pinned host minibatches; losses read back"
    return {"value": round(n_upd * B * world / (total_ms / 1e3), 2), "unit": "samples/s",
            "h2d_bytes_per_step": B * per * 4, "d2h_bytes_per_step": 8 // nb if pair else 8,
            "path": path}


def run_actor(args, rank, world, workload):
    """configs[4]: actor forward + BPTT + gradient allreduce over the rank's shard of the 65 536-row
    global batch (strong scaling); configs[0]: the fp32 actor forward + backward at B = 100 per rank
    (weak scaling). The step is captured as one CUDA graph (NCCL call included) unless --eager."""
    import numpy as np
    import torch
    import synthgen as sg
    import paper_2502_17496_b200 as pk
    from paper_2502_17496_b200 import _lib
    shape, _, Bg = sg.preset(workload)
    strong = workload == "cfg4"
    B = Bg // world if strong else Bg
    actor = pk.SpikingActor(pk.actor_cfg_from(shape, engine=args.engine), B)
    rng = np.random.default_rng(0)
    actor.load(sg.actor_params(shape, rng))
    comm = pk.Comm(rank, world) if (world > 1 or FORCE_COMM) else None
    if comm:
        comm.broadcast(actor.params)
        actor.refresh()
    g = torch.Generator(device="cuda").manual_seed(rank)
    obs = torch.clamp(torch.randn(B, shape.obs_dim, device="cuda", generator=g), -5, 5)
    ga = torch.randn(B, shape.act_dim, device="cuda", generator=g)

    def step_on(o, g):
        actor.forward(o)
        actor.backward(o, g, comm=comm)   # with comm: bucketed gradient mean overlapping the BPTT

    def step(k=0):
        step_on(obs, ga)

    lib = pk.lib()
    step()                          # first launches (module loading, tensor maps) outside the profile
    summ = _profile_pass(step)
    overlap = comm_overlap(_LAST_TIMELINE) if comm else None
    dom = max(summ, key=lambda e: e["total_ms"])["name"]
    lib.spikerl_launch_count(1)
    step()
    n_launch = lib.spikerl_launch_count(1)
    watch = _lib.Watch(dom, 16)
    wgraph = None
    if args.eager:
        def run(k):
            watch.arm()
            step(k)
        per = None
    else:
        # as for TD3: the value is timed on the plain graph, the dominant kernel live on a second
        # capture with event nodes around its launches, replayed for as many steps
        watch.arm()
        wgraph = _capture(step)
        per = watch.used()
        _lib.Watch.off()
        graph = _capture(step)

        def run(k):
            graph.replay()
    for k in range(args.warmup):
        run(k)
    torch.cuda.synchronize()
    flush = None if (strong or args.no_flush) else torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def after(k):
        torch.cuda.synchronize()
        watch.collect(per if per is not None else watch.used())
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    if wgraph is None:
        total_ms = time_steps(run, args.steps, flush, world, after_step=after)
    else:
        total_ms = time_steps(run, args.steps, flush, world)
        wgraph.replay()   # its first replay (upload) outside its timed loop
        torch.cuda.synchronize()
        time_steps(lambda k: wgraph.replay(), args.steps, flush, world, after_step=after)
    clocks = clk.stop()
    _lib.Watch.off()
    secs = total_ms / 1e3
    gsum = Bg if strong else B * world
    out = {"metric": METRIC, "value": round(args.steps * gsum / secs, 2), "unit": "samples/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
           "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
           "dtype": "bf16" if shape.precision == "bf16" else "f32",
           "data": "synthetic observations ~N(0,1) clipped +-5, upstream grads ~N(0,1)",
           "config": {"workload": f"{workload}: spiking actor fwd+BPTT (+allreduce), obs {shape.obs_dim} act "
                                  f"{shape.act_dim} pop 10/10 hidden {shape.n1}-{shape.n2} T={shape.T} "
                                  f"{shape.precision}", "global_batch": gsum, "per_rank_batch": B,
                      "parallelism": f"dp{world}", "engine": args.engine,
                      "cuda_graph": not args.eager,
                      "l2": "inputs and tape (GBs) exceed L2" if strong else
                      ("flushed between timed steps (256 MB read, outside the events)" if flush is not None
                       else "not flushed")},
           "clocks": clocks, "gpu_launches": int(n_launch) * args.steps}
    en = energy_window(run, clk)
    if en:
        en["joules_per_step"] = round(en["joules"] / en["steps"], 5)
        en["samples_per_joule"] = round(en["steps"] * gsum / max(en["joules"], 1e-9), 1)
        out["energy"] = en
    out["roofline"] = dominant_kernel(summ, peaks(), (watch.launches, watch.total_ms), total_ms, workload,
                                      long_step=strong,
                                      clocks=clocks)
    out["kernel_breakdown"] = _breakdown(summ)
    if strong:
        out["hbm_kernels"] = hbm_kernels(actor, summ)
    if overlap:
        out["comm_overlap"] = overlap
    if not args.no_e2e:
        out["e2e"] = e2e_actor(args, world, actor, step_on, obs, ga, gsum, shape)
    return out


def comm_overlap(tl):
    """Timeline of the profiling pass (events on each launch's own stream): for each gradient bucket's
    allreduce (comm stream), its interval and the compute kernels whose intervals overlap it."""
    out = []
    for name, a, b in tl:
        if not name.startswith("allreduce_bucket"):
            continue
        ov = [(n2, round(min(b, b2) - max(a, a2), 4)) for n2, a2, b2 in tl
              if not n2.startswith("allreduce") and min(b, b2) > max(a, a2)]
        out.append({"bucket": name[len("allreduce_bucket_"):], "start_ms": round(a, 4), "end_ms": round(b, 4),
                    "overlapped_by": ov})
    return out


def e2e_actor(args, world, actor, step_on, obs, ga, gsum, shape):
    """End to end through the public API: every step copies its observations and upstream action
    gradients from pinned host memory and reads the parameter gradients back into pinned host
    memory. Graphs (two, alternating device input buffers) of [H2D of the NEXT step's inputs on a
    copy stream || forward -> backward (-> allreduce) on this step's -> D2H of the gradients]: the
    input copies overlap the previous step's compute (every step's copy is inside the timed region
    except the first, made before it)."""
    import torch
    host_obs = obs.cpu().pin_memory()
    host_ga = ga.cpu().pin_memory()
    grads_host = torch.empty(actor.n_params, dtype=torch.float32).pin_memory()
    ins = [(obs, ga), (obs.clone(), ga.clone())]

    def h2d(i):
        ins[i][0].copy_(host_obs, non_blocking=True)
        ins[i][1].copy_(host_ga, non_blocking=True)

    if args.eager:
        def run(k):
            h2d(0)
            step_on(*ins[0])
            grads_host.copy_(actor.grads, non_blocking=True)
    else:
        graphs = []
        cs, cp = torch.cuda.Stream(), torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            for i in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    cp.wait_stream(cs)
                    with torch.cuda.stream(cp):
                        h2d(1 - i)
                    step_on(*ins[i])
                    cs.wait_stream(cp)
                    grads_host.copy_(actor.grads, non_blocking=True)
                graphs.append(g)
        torch.cuda.current_stream().wait_stream(cs)
        h2d(0)
        torch.cuda.synchronize()
        run = lambda k: graphs[k % 2].replay()
    n = max(4, args.steps // 2)
    n += n % 2
    for k in range(2 * max(1, args.warmup // 4)):
        run(k)
    total = time_steps(run, n, None, world)
    B = obs.shape[0]
    return {"value": round(n * gsum / (total / 1e3), 2), "unit": "samples/s",
            "h2d_bytes_per_step": B * (shape.obs_dim + shape.act_dim) * 4, "d2h_bytes_per_step": actor.n_params * 4,
            "path": ("graphs" if not args.eager else "eager") + " of [H2D of the next step's obs + upstream grads from "
                    "pinned host on a copy stream || spikerl_actor_forward -> spikerl_actor_backward (-> allreduce) "
                    "on this step's -> D2H of the gradients] (double-buffered inputs)"}


def hbm_kernels(actor, summ, reps=20):
    """The HBM-bound kernels of the path against the measured copy bandwidth (north_star: LIF scans
    and Adam >= 70%): the output-layer reverse scan from the step's launch list, and Adam / Polyak
    over the configs[4] actor's 5.08 M parameters (28 / 12 algorithmic bytes per parameter), each
    launch timed alone with CUDA events on its stream, L2 flushed between launches."""
    import torch
    import paper_2502_17496_b200 as pk
    pk_peaks = peaks()
    res = {}
    for e in summ:
        if e["name"] == "dec_bwd_outscan":
            gbs = e["bytes"] / (e["total_ms"] / 1e3) / 1e9
            res["dec_bwd_outscan"] = {"achieved": round(gbs, 1), "unit": "GB/s", "peak": pk_peaks["hbm_gbs"],
                                      "frac": round(gbs / pk_peaks["hbm_gbs"], 4),
                                      "bytes_per_launch": e["bytes"] / e["launches"],
                                      "us_per_launch": round(e["total_ms"] / e["launches"] * 1e3, 2)}
    n = actor.n_params
    f32 = dict(dtype=torch.float32, device="cuda")
    p = actor.params.clone()
    g = torch.randn(n, **f32) * 1e-3
    m, v = torch.zeros(n, **f32), torch.zeros(n, **f32)
    t = torch.zeros(2, dtype=torch.int64, device="cuda")
    tgt = p.clone()
    flush = torch.empty(64 * 1024 * 1024, **f32)
    for name, bpp, fn in (("adam", 28.0, lambda: pk.adam(p, g, m, v, t, 1e-4)),
                          ("polyak", 12.0, lambda: pk.polyak(tgt, p, 0.005))):
        fn()
        tot = 0.0
        for _ in range(reps):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        us = tot / reps * 1e3
        gbs = bpp * n / (us / 1e6) / 1e9
        res[name] = {"achieved": round(gbs, 1), "unit": "GB/s", "peak": pk_peaks["hbm_gbs"],
                     "frac": round(gbs / pk_peaks["hbm_gbs"], 4), "bytes_per_launch": bpp * n,
                     "us_per_launch": round(us, 2), "params": n}
    # the standalone forward-scan ablation (SURVEY D-2) at the configs[4] hidden-layer size: reads the
    # fp32 currents [T][B][N] the fused FWD epilogue never writes, writes the spike / window planes
    T, B, N = actor.cfg.T, actor.batch, actor.cfg.hidden2
    W = (N + 31) // 32
    cur = torch.randn(T * B * N, **f32) * 0.5
    planes = torch.zeros(2, T * B * W, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream

    def scan():
        rc = pk.lib().spikerl_lif_scan_forward(cur.data_ptr(), T, B, N, actor.cfg.d_c, actor.cfg.d_v, actor.cfg.v_th,
                                               actor.cfg.surr_window, planes[0].data_ptr(), planes[1].data_ptr(),
                                               stream)
        assert rc == 0, rc
    scan()
    tot = 0.0
    for _ in range(reps // 4):
        l2_flush(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        scan()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    us = tot / (reps // 4) * 1e3
    nbytes = float(T) * B * (4 * N + 8 * W)
    gbs = nbytes / (us / 1e6) / 1e9
    res["lif_scan_ablation"] = {"achieved": round(gbs, 1), "unit": "GB/s", "peak": pk_peaks["hbm_gbs"],
                                "frac": round(gbs / pk_peaks["hbm_gbs"], 4), "bytes_per_launch": nbytes,
                                "us_per_launch": round(us, 2), "shape": [T, B, N],
                                "what": "standalone forward LIF scan over fp32 currents (the ablation of the "
                                        "fused FWD epilogue, which never writes them)"}
    del cur, planes
    return res


def main():
    args = parse()
    if args.impl == "reference":
        return reference(args)
    import torch
    rank, world, local = dist_init(args)
    if args.workload in ("cfg0", "cfg4"):
        out = run_actor(args, rank, world, args.workload)
        if args.workload == "cfg4" and not args.no_td3_extra:
            # configs[3] at per-rank batch 4096: the TD3 updates/s throughput regime (weak scaling)
            td = run_td3(args, rank, world, "cfg3L")
            td.pop("metric", None)
            out["td3"] = td
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_actor(args.workload, B_sample=16 if args.workload == "cfg4" else 100)
            # the oracle on one host core as well (SURVEY D-5), a shorter sample
            out["cpu_baseline"]["single_thread"] = cpu_baseline_actor(
                args.workload, B_sample=16 if args.workload == "cfg4" else 100, seconds=5.0, threads=1)
            out["gps_up"] = gps_up(out["value"], out.get("energy"), out["cpu_baseline"])
    else:
        out = run_td3(args, rank, world, args.workload)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_td3(args.workload)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def reference(args):
    """The oracle, as it stands, on the host cores: same metric/unit/config as our arm. Exactly
    --warmup untimed steps, then up to --steps timed steps (stops early at a time budget and says so)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synthgen as sg
    name = args.workload
    shape, cs, B = sg.preset(name)
    rng = np.random.default_rng(0)
    if name in ("cfg0", "cfg4"):
        p = sg.actor_params(shape, rng)
        Bs = 8 if name == "cfg4" else B

        def step(k):
            s = sg.observations(rng, Bs, shape.obs_dim)
            a, tape = oracle.actor_forward(p, shape, s)
            oracle.actor_backward(p, shape, tape, sg.action_grads(rng, Bs, shape.act_dim))
        per_step = Bs
        sample = (f"each step = {Bs} rows of cfg4 actor fwd+BPTT (value extrapolates linearly in B)" if name == "cfg4"
                  else f"each step = the full cfg0 batch of {B} rows, actor fwd+BPTT")
    else:
        st = [oracle.init_state(sg.actor_params(shape, rng), sg.critic_params(cs, rng), sg.critic_params(cs, rng))]
        hp = sg.TD3Hyper()

        def step(k):
            st[0], _ = oracle.td3_update(st[0], shape, cs, hp, sg.replay_batch(rng, B, shape.obs_dim, shape.act_dim),
                                         sg.target_noise(rng, B, shape.act_dim), k + 1)
        per_step, sample = B, f"each step = one full TD3 update of {name} at B={B}"
    budget = 150.0
    t_start = time.time()
    for k in range(args.warmup):
        step(k)
    t0 = time.time()
    done = 0
    for k in range(args.steps):
        step(args.warmup + k)
        done += 1
        if time.time() - t_start > budget:
            break
    dt = time.time() - t0
    v = done * per_step / dt
    cores = len(os.sched_getaffinity(0))
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "samples/s", "n_gpus": args.gpus,
           "steps": done, "warmup": args.warmup, "ms_per_step": round(dt / done * 1e3, 3),
           "higher_is_better": True, "scaling": "weak" if name not in ("cfg4",) else "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "config": {"workload": name, "per_rank_batch": B},
           "cpu_baseline": {"value": round(v, 3), "unit": "samples/s", "cores": cores, "kind": "oracle",
                            "sample": sample + (f"; stopped after {done} of {args.steps} steps (time budget)"
                                                if done < args.steps else "")},
           "e2e": {"value": round(v, 3), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
