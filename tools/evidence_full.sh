#!/bin/bash
# tools/evidence.sh, then the ncu summaries written on the box (the .ncu-rep files exceed what a
# gpurun call brings back): profiles/ outputs copied to gpurun_out/newprof/, reports deleted.
set -u
O=gpurun_out
bash tools/evidence.sh
python tools/ncu_summarize.py r01_cfg4 $O/launches_cfg4.csv lif_fwd_tc_L1=$O/prof_fwd1.ncu-rep \
  lif_fwd_tc_L2=$O/prof_fwd2.ncu-rep lif_dw_tc_L1=$O/prof_dw1.ncu-rep lif_dx_tc_L2=$O/prof_dx2.ncu-rep \
  lif_dx_tc_L3=$O/prof_dx3.ncu-rep enc_fwd=$O/prof_enc_fwd.ncu-rep dec_bwd_outscan=$O/prof_dec_bwd_outscan.ncu-rep \
  adam=$O/prof_adam_kernel.ncu-rep polyak=$O/prof_polyak_kernel.ncu-rep > $O/summ4.log 2>&1; echo "summ4 rc=$?"
python tools/ncu_summarize.py r01_cfg1 $O/launches_cfg1.csv > $O/summ1.log 2>&1; echo "summ1 rc=$?"
python tools/ncu_hot.py $O/prof_fwd1.ncu-rep 20 > $O/hot_fwd1.txt 2>&1
mkdir -p $O/newprof; cp profiles/r01_cfg*_ncu_summary.md profiles/ncu_traffic.json $O/newprof/
ls /sys/class/powercap/ > $O/powercap.txt 2>&1
rm -f $O/prof_*.ncu-rep
