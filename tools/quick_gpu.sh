#!/bin/bash
# one GPU call: gpu tests, then the cfg4 and cfg1 bench lines (kernel breakdown printed)
set -u
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gputests.log
python bench.py --workload cfg4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1 rc=$?"
python - <<'PY'
import json
for f in ("cfg4", "cfg1"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{f}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no line", e); continue
    print(f, "ms/step", d["ms_per_step"], "value", d["value"], "roofline", d["roofline"]["kernel"], d["roofline"]["frac"])
    print("  ", " ".join(f"{k['name']}={k['total_ms']:.3f}" for k in d["kernel_breakdown"]))
    if d.get("hbm_kernels"):
        print("  ", {k: v["frac"] for k, v in d["hbm_kernels"].items()})
PY
