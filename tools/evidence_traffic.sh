#!/bin/bash
# One GPU call: ncu --set full captures of the dominant kernel of every bench line other than
# configs[4] (whose captures tools/evidence.sh takes), at that line's own workload, so that
# roofline.traffic (profiles/ncu_traffic.json, keyed "<workload>:<kernel>") is the DRAM traffic of
# the same launch shape the line times. Summarised here by tools/ncu_summarize.py.
set -u
O=gpurun_out
python tools/kernel_times.py cfg3L 4096 1 > $O/plain_kt3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"tc_kernel<\\(int\\)0," -s 2 -c 1 -o $O/prof_cfg3L_fwd1 \
      python tools/kernel_times.py cfg3L 4096 1 > $O/ncu_cfg3L_fwd1.log 2>&1
for w in cfg1 cfg2 cfg3s; do
  python tools/td3_launches.py $w 2 > $O/plain_$w.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:critic_fwd_mma -s 2 -c 1 \
        -o $O/prof_${w}_cfwd python tools/td3_launches.py $w 2 > $O/ncu_${w}_cfwd.log 2>&1
done
python tools/kernel_times.py cfg0 100 1 > $O/plain_kt0.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:enc_grad -s 2 -c 2 \
      -o $O/prof_cfg0_encgrad python tools/kernel_times.py cfg0 100 1 > $O/ncu_cfg0_encgrad.log 2>&1
for r in $O/prof_cfg3L_fwd1 $O/prof_cfg1_cfwd $O/prof_cfg2_cfwd $O/prof_cfg3s_cfwd $O/prof_cfg0_encgrad; do
  bash tools/ncu_export.sh $r.ncu-rep
done
ls -la $O | grep prof_
