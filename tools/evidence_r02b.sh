# r02 late evidence: cfg1 / cfg2 launch lists and ncu --set full of the new critic kernels
O=gpurun_out
for w in cfg1 cfg2; do
  python tools/td3_launches.py $w 2 > $O/plain_$w.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv \
        python tools/td3_launches.py $w 2 > $O/ncu_l_$w.log 2>&1
  echo "$w launches rc=$?"
done
for spec in critic_actor_fused:cfg1 critic_adam_kernel:cfg1 critic_update_fused:cfg2; do
  IFS=: read k w <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/prof_${k}_$w \
      python tools/td3_launches.py $w 3 > $O/ncu_${k}.log 2>&1
  echo "$k rc=$?"
  bash tools/ncu_export.sh $O/prof_${k}_$w.ncu-rep
done
ls -la $O | tail -20
