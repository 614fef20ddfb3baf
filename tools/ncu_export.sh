#!/bin/bash
# On the GPU box: export the raw / details / source (SASS) pages of ncu reports as gzipped CSV next
# to them and delete the reports (gpurun brings back at most 64 MiB; a full tcgen05 report is ~15 MB).
for rep in "$@"; do
  base=${rep%.ncu-rep}
  ncu -i $rep --page raw --csv | gzip > $base.raw.csv.gz
  ncu -i $rep --page details --csv | gzip > $base.details.csv.gz
  ncu -i $rep --page source --csv --print-source sass | gzip > $base.source.csv.gz
  rm -f $rep
done
