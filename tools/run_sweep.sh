timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_critic or critic" > gpurun_out/t_fused.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/t_fused.log
for w in cfg3s cfg1 cfg2; do
bash tools/ab_env2.sh $w "SPIKERL_X=new" "SPIKERL_LIB_PATH=ab/libspikerl_base.so" 2
done
