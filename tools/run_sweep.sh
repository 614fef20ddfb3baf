timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_critic or pair_matches" > gpurun_out/t_fused.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/t_fused.log
bash tools/ab_env2.sh cfg1 "SPIKERL_CRITIC_FUSED_U2=1" "SPIKERL_CRITIC_FUSED_U2=0" 2
bash tools/ab_env2.sh cfg3s "SPIKERL_CRITIC_FUSED_U2=1" "SPIKERL_CRITIC_FUSED_U2=0" 2
