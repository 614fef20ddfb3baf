#!/bin/bash
# A/B per-kernel times of two library builds (ab/lib_head.so vs the in-tree build), alternating.
O=gpurun_out
for r in 1 2; do
  for L in ab/lib_head.so paper_2502_17496_b200/libspikerl.so; do
    echo "== $L round $r"
    for w in ${AB_CFGS:-cfg4 cfg3L cfg1}; do
      SPIKERL_LIB_PATH=$PWD/$L python tools/kernel_times.py $w 2>&1 | grep -E "${AB_PAT:-fwd|dx|enc|sum}"
    done
  done
done
