set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_critic" > gpurun_out/t_fused.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/t_fused.log
bash tools/ab_env2.sh cfg1 "SPIKERL_OUTSCAN_IN_CRITIC=1" "SPIKERL_OUTSCAN_IN_CRITIC=0" 2
bash tools/ab_env2.sh cfg3s "SPIKERL_OUTSCAN_IN_CRITIC=1" "SPIKERL_OUTSCAN_IN_CRITIC=0" 1
