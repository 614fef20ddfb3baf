#!/bin/bash
# Diagnostics: per-kernel times of one cfg4 step with parts of the tcgen05 engine disabled
# (SPIKERL_TC_DBG bits: 1 expanders skip smem stores, 2 epilogue skipped, 4 MMAs skipped).
# Results are wrong by construction in the ablated runs; only the timings mean anything.
for d in ${@:-0 1 2 4 3 6 7}; do
  SPIKERL_TC_DBG=${d%%:*} SPIKERL_TC_TT=${d#*:} timeout 120 python bench.py --workload cfg4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg=$d', d['ms_per_step'], ' '.join(f\"{k['name']}={k['total_ms']:.3f}\" for k in d['kernel_breakdown']))"
done
