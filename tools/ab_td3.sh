#!/bin/bash
# A/B of the TD3 bench line between ab/lib_head.so and the in-tree build, alternating (same box).
for r in 1 2 3; do
  for L in ab/lib_head.so paper_2502_17496_b200/libspikerl.so; do
    for w in ${AB_CFGS:-cfg1 cfg3L}; do
      v=$(SPIKERL_LIB_PATH=$PWD/$L python bench.py --workload $w --steps 200 --warmup 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])")
      echo "$w $(basename $L) r$r ms/update=$v"
    done
  done
done
