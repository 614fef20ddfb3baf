set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_critic" > gpurun_out/t_fused.log 2>&1; echo "fused test rc=$?"; tail -3 gpurun_out/t_fused.log
for w in cfg1 cfg3s cfg2; do
  for v in "SPIKERL_CRITIC_ACT_FUSED=1" "SPIKERL_CRITIC_ACT_FUSED=0"; do
    env $v timeout 300 python bench.py --workload $w --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2> gpurun_out/b.err; echo "$w [$v] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step']*1000,'us')" 2>&1)"
  done
done
for v in "SPIKERL_CRITIC_ADAM_TILED=1" "SPIKERL_CRITIC_ADAM_TILED=0"; do
  env $v timeout 300 python bench.py --workload cfg3L --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2> gpurun_out/b.err; echo "cfg3L [$v] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step']*1000,'us')" 2>&1)"
done
