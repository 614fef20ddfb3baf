#!/bin/bash
# One GPU call that regenerates this round's evidence under gpurun_out/ (summarised into profiles/
# by tools/ncu_summarize.py on the CPU box): the driver's default bench line (configs[4] + the
# configs[3] B=4096 TD3 keys), bench lines of the other workloads, the reference arm, cold launch
# lists (configs[4] step, configs[1] / configs[3] B=4096 update pairs) and ncu --set full captures.
set -u
O=gpurun_out
PART=${EVIDENCE_PART:-all}
if [ "$PART" != "ncu" ]; then
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
python bench.py --workload cfg0 --steps 200 --warmup 20 > $O/bench_cfg0.json 2> $O/bench_cfg0.err; echo "cfg0 rc=$?"
python bench.py --workload cfg1 --steps 200 --warmup 20 > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "cfg1 rc=$?"
for w in cfg2 cfg3s cfg3L; do
  python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"
done
python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_default.json 2> $O/ref_default.err; echo "ref rc=$?"
python bench.py --impl reference --workload cfg1 --steps 5 --warmup 1 > $O/ref_cfg1.json 2> $O/ref_cfg1.err; echo "ref1 rc=$?"
fi
if [ "$PART" != "bench" ]; then
# launch lists (cold, serialised: shares only)
python tools/kernel_times.py cfg4 65536 1 > $O/plain4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
      python tools/kernel_times.py cfg4 65536 1 > $O/ncu_l4.log 2>&1
for w in cfg1 cfg3L; do
  python tools/td3_launches.py $w 2 > $O/plain_$w.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
        python tools/td3_launches.py $w 2 > $O/ncu_l_$w.log 2>&1
done
# full captures of the configs[4] hot kernels (one step of kernel_times: warm step, then the profiled one)
for spec in fwd1:0:2 fwd2:0:3 dw1:3:5 dx2:1:3 dx3:1:2 enc:2:1; do
  IFS=: read name mode skip <<< "$spec"
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"tc_kernel<\\(int\\)$mode," -s $skip -c 1 -o $O/prof_$name \
      python tools/kernel_times.py cfg4 65536 1 > $O/ncu_$name.log 2>&1
  bash tools/ncu_export.sh $O/prof_$name.ncu-rep
done
for k in enc_fwd dec_bwd_outscan; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/prof_$k \
      python tools/kernel_times.py cfg4 65536 1 > $O/ncu_$k.log 2>&1
  bash tools/ncu_export.sh $O/prof_$k.ncu-rep
done
# the tcgen05 critic at configs[3] B = 4096 (CF1 / CF2 / CB1 modes)
for spec in cf1:6 cf2:7 cb1:8; do
  IFS=: read name mode <<< "$spec"
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"tc_kernel<\\(int\\)$mode," -s 4 -c 1 -o $O/prof_$name \
      python tools/td3_launches.py cfg3L 2 > $O/ncu_$name.log 2>&1
  bash tools/ncu_export.sh $O/prof_$name.ncu-rep
done
python tools/small_kernels.py > $O/small.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:adam_kernel -s 95 -c 1 -o $O/prof_adam_kernel \
    python tools/small_kernels.py > $O/ncu_adam.log 2>&1
bash tools/ncu_export.sh $O/prof_adam_kernel.ncu-rep
fi
du -sh $O; ls -la $O
