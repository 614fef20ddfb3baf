set -u
python tools/graph_timeline.py cfg1 > gpurun_out/tl_cfg1.txt 2>&1; echo "tl rc=$?"
SPIKERL_TD3_SERIAL=1 python tools/graph_timeline.py cfg1 > gpurun_out/tl_cfg1_serial.txt 2>&1; echo "tls rc=$?"
python tools/td3_phase_timing.py cfg1 > gpurun_out/phase_cfg1.txt 2>&1; echo "ph rc=$?"
