#!/bin/bash
# ncu --set full captures of single tcgen05 launches of one cfg4 step; run only after
# tools/profile_cfg4.sh has exited 0 on the same build.
#   tools/profile_cfg4_tc.sh <name>:<mode>:<skip> ...   (mode 0 FWD, 1 DX, 2 ENC, 3 DW; skip = index
#   of the launch of that mode within the step, e.g. fwd2:0:1 = FWD of layer 2, dx3:1:0 = DX L3)
for spec in "${@:-fwd1:0:0 dw1:3:2}"; do
  IFS=: read name mode skip <<< "$spec"
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"tc_kernel<\\(int\\)$mode" -s $skip -c 1 -o gpurun_out/prof_$name \
      bash tools/profile_cfg4.sh > gpurun_out/ncu_$name.log 2>&1
done
