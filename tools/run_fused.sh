set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_critic or td3_two or teacher or schedule_independent" > gpurun_out/t_fused.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/t_fused.log
timeout 900 python -m pytest tests/test_gpu_td3_parity.py -x -q > gpurun_out/t_td3p.log 2>&1; echo "td3 parity rc=$?"; tail -3 gpurun_out/t_td3p.log
for w in cfg1 cfg3s cfg2; do
  for v in "SPIKERL_X=1"; do
    env $v timeout 300 python bench.py --workload $w --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2> gpurun_out/b.err; echo "$w [$v] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step']*1000,'us')" 2>&1)"
  done
done
