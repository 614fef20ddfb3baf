# A/B of two environment settings on one box, alternating: bash tools/ab_env2.sh <workload> "<envA>" "<envB>" [rounds]
w=$1; A=$2; Bv=$3; n=${4:-3}
for i in $(seq $n); do
  for v in "$A" "$Bv"; do
    env $v timeout 300 python bench.py --workload $w --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
    echo "$w [$v] $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1000,2),'us')" 2>&1)"
  done
done
