for c in "cfg1 256" "cfg2 512" "cfg3s 100" "cfg3L 4096"; do
  for e in "" "SPIKERL_TC_PAIR=0"; do
    echo "== $c [$e]"; env $e python tools/kernel_times.py $c 20 2>&1 | grep "tc\|sum"
  done
done
