SPIKERL_CRITIC_FUSED=1 python tools/fused_trace.py cfg1 9
bash tools/ab_env2.sh cfg1 "SPIKERL_CRITIC_FUSED=1" "SPIKERL_CRITIC_FUSED=0" 2
