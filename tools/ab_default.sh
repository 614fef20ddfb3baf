#!/bin/bash
# A/B of the default bench line (configs[4] step) between ab/lib_head.so and the in-tree build,
# alternating on one box; prints ms/step and the DW kernels' totals of each run.
for r in $(seq ${AB_R:-3}); do
  for L in ab/lib_head.so paper_2502_17496_b200/libspikerl.so; do
    SPIKERL_LIB_PATH=$PWD/$L python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $L)', 'r$r', d['ms_per_step'], ' '.join(f\"{k['name']}={k['total_ms']:.3f}\" for k in d['kernel_breakdown'] if 'dw' in k['name']))"
  done
done
