#!/bin/bash
# Diagnostics: per-kernel times (tools/kernel_times.py) of the cfg4 actor step with parts of the
# tcgen05 engine disabled (SPIKERL_TC_DBG bits: 1 expanders skip smem stores, 2 epilogue skipped,
# 4 MMAs skipped, 8 DW expanders skip loads, 16 TMA producer skips loads). Wrong results by design.
for d in ${@:-0 2 4 6 1 16 17 20 22}; do
  echo "dbg=$d $(SPIKERL_TC_DBG=$d timeout 300 python tools/kernel_times.py cfg4 65536 2 2>/dev/null | grep -E 'lif_|enc_grad' | awk '{printf "%s=%s ", $1, $2}')"
done
