#!/bin/bash
# ncu --set full captures of the two largest tcgen05 launches of one cfg4 step (FWD L1, DW L1);
# run only after tools/profile_cfg4.sh has exited 0 on the same build.
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc_kernel<\\(int\\)0" -s 0 -c 1 -o gpurun_out/prof_fwd1 bash tools/profile_cfg4.sh > gpurun_out/ncu_fwd1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc_kernel<\\(int\\)3" -s 2 -c 1 -o gpurun_out/prof_dw1 bash tools/profile_cfg4.sh > gpurun_out/ncu_dw1.log 2>&1
