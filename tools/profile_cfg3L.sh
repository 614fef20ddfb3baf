#!/bin/bash
# a short cfg3L TD3 bench run for ncu captures (the eager profiling pass launches every kernel)
exec python bench.py --workload cfg3L --steps 4 --warmup 3 --no-e2e --no-cpu-baseline
