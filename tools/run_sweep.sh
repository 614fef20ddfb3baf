timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_critic" > gpurun_out/t_fused.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/t_fused.log
timeout 900 python -m pytest tests/test_gpu_td3_parity.py -x -q > gpurun_out/t_td3p.log 2>&1; echo "td3 parity rc=$?"; tail -1 gpurun_out/t_td3p.log
SPIKERL_CRITIC_FUSED=1 python tools/fused_trace.py cfg1 9
bash tools/ab_env2.sh cfg2 "SPIKERL_X=new" "SPIKERL_LIB_PATH=ab/libspikerl_base.so" 2
bash tools/ab_env2.sh cfg1 "SPIKERL_CRITIC_FUSED=1" "SPIKERL_CRITIC_FUSED=0" 2
bash tools/ab_env2.sh cfg1 "SPIKERL_X=new" "SPIKERL_LIB_PATH=ab/libspikerl_base.so" 1
