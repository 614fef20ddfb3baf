#!/bin/bash
# A/B of the TD3 bench lines under an environment switch: AB_ENV="VAR=value" vs unset, alternating.
for r in 1 2; do
  for w in ${AB_CFGS:-cfg1 cfg2 cfg3s}; do
    for e in "" "$AB_ENV"; do
      v=$(env $e python bench.py --workload $w --steps 200 --warmup 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])")
      echo "$w [${e:-default}] r$r $v"
    done
  done
done
