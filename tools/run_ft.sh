SPIKERL_CRITIC_FUSED_G=148 python tools/fused_trace.py cfg1 9
SPIKERL_CRITIC_FUSED_G=148 SPIKERL_CRITIC_FUSED_DBG=8 python tools/fused_trace.py cfg1 9
SPIKERL_CRITIC_FUSED_G=148 python tools/fused_trace.py cfg3s 9
