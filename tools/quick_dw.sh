# DW epilogue / reduction A/B (ab/lib_head.so vs in-tree): per-kernel times, TD3 lines, default line
for L in ab/lib_head.so paper_2502_17496_b200/libspikerl.so; do
for c in "cfg1 256" "cfg3L 4096"; do echo "== $L $c"; SPIKERL_LIB_PATH=$PWD/$L python tools/kernel_times.py $c 20 2>&1 | grep "dw\|sum"; done
echo "== $L cfg4"; SPIKERL_LIB_PATH=$PWD/$L python tools/kernel_times.py cfg4 65536 3 2>&1 | grep "dw\|sum"
done
AB_CFGS="${AB_CFGS:-cfg1 cfg2 cfg3s cfg3L}" bash tools/ab_td3.sh > gpurun_out/abt.log 2>&1
