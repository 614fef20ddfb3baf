O=gpurun_out
python tools/td3_launches.py cfg1 3 > $O/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:critic_update_fused -s 2 -c 1 -o $O/prof_fused python tools/td3_launches.py cfg1 3 > $O/ncu_fused.log 2>&1
ncu -i $O/prof_fused.ncu-rep --page details --csv > $O/prof_fused.details.csv
ncu -i $O/prof_fused.ncu-rep --page raw --csv | gzip > $O/prof_fused.raw.csv.gz
ncu -i $O/prof_fused.ncu-rep --page source --csv --print-source sass | gzip > $O/prof_fused.source.csv.gz
rm -f $O/prof_fused.ncu-rep
tail -3 $O/ncu_fused.log
