#!/bin/bash
# One GPU call that regenerates this round's evidence under gpurun_out/ (summarised into profiles/
# by tools/ncu_summarize.py on the CPU box): bench lines for every workload, the reference arm,
# the cold launch lists of cfg1 / cfg4 and ncu --set full captures of the cfg4 hot kernels.
set -u
O=gpurun_out
python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "cfg1 rc=$?"
python bench.py --workload cfg4 --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4 rc=$?"
for w in cfg2 cfg3s cfg3L; do
  python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"
done
python bench.py --impl reference --steps 5 --warmup 1 > $O/ref_cfg1.json 2> $O/ref_cfg1.err; echo "ref rc=$?"
# launch lists (cold, serialised: shares only)
bash tools/profile_cfg1.sh > $O/plain1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1.csv bash tools/profile_cfg1.sh > $O/ncu_l1.log 2>&1
bash tools/profile_cfg4.sh > $O/plain4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv bash tools/profile_cfg4.sh > $O/ncu_l4.log 2>&1
# full captures: FWD L1, DW L1, DX L2, enc_fwd, outscan, adam (the HBM kernels run by bench's hbm_kernels)
bash tools/profile_cfg4_tc.sh fwd1:0:0 fwd2:0:1 dw1:3:2 dx2:1:1 dx3:1:0
for k in enc_fwd dec_bwd_outscan adam_kernel polyak_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/prof_$k bash tools/profile_cfg4.sh > $O/ncu_$k.log 2>&1
done
ls -la $O
