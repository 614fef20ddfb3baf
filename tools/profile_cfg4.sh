#!/bin/bash
# one cfg4 actor fwd+BPTT step (B=65536) for ncu captures
exec python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
