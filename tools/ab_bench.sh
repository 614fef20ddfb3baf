#!/bin/bash
# A/B timing of two builds of libspikerl.so on one box (diagnostics): alternates the variants
# paper_2502_17496_b200/libspikerl_{A,B}.so, N rounds of `bench.py --workload W`, and prints the
# per-kernel times of every run. Usage: tools/ab_bench.sh <workload> <rounds>
W=${1:-cfg4}; N=${2:-3}
L=paper_2502_17496_b200
cp $L/libspikerl.so /tmp/libspikerl_cur.so
for r in $(seq $N); do
  for v in A B; do
    cp $L/libspikerl_$v.so $L/libspikerl.so
    python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], ' '.join(f\"{k['name']}={k['total_ms']:.3f}\" for k in d['kernel_breakdown']))"
  done
done
cp /tmp/libspikerl_cur.so $L/libspikerl.so
