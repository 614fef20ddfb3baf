#!/bin/bash
# cfg1 / cfg3L TD3 bench under the scheduling switches: default, no PDL, one stream, both
for w in ${MODES_CFGS:-cfg1 cfg3L}; do
  for env in "" "SPIKERL_PDL=0" "SPIKERL_TD3_SERIAL=1" "SPIKERL_PDL=0 SPIKERL_TD3_SERIAL=1"; do
    r=$(env $env python bench.py --workload $w --steps 100 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])")
    echo "$w [$env] ms/update=$r"
  done
done
