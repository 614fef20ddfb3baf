#!/bin/bash
# A/B of the TD3 bench lines under several environment settings, alternating on one box:
# AB_ENVS="VAR=a VAR=b ..." (each against the default), AB_CFGS (default cfg1 cfg2 cfg3s), AB_R rounds.
for r in $(seq ${AB_R:-2}); do
  for w in ${AB_CFGS:-cfg1 cfg2 cfg3s}; do
    for e in "" $AB_ENVS; do
      v=$(env $e python bench.py --workload $w --steps 200 --warmup 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])")
      echo "$w [${e:-default}] r$r $v"
    done
  done
done
