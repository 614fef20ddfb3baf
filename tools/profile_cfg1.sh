#!/bin/bash
# a short cfg1 TD3 bench run for ncu captures (eager profiling pass launches every kernel)
exec python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline
