#!/bin/bash
# One GPU call: GPU tests (pytest -k "$QK" if set, else all), cfg4 per-kernel times, and the cfg3L /
# cfg1 / default bench lines in short runs (no e2e / cpu baseline). Summary on stdout.
set -u
O=gpurun_out
if [ -n "${QK:-}" ]; then timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$QK" > $O/gputests.log 2>&1
else timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gputests.log 2>&1; fi
echo "tests rc=$?"; tail -2 $O/gputests.log
python tools/kernel_times.py cfg4 65536 3 > $O/kt4.log 2>&1; cat $O/kt4.log
python tools/kernel_times.py cfg3L 4096 5 > $O/kt3.log 2>&1; cat $O/kt3.log
python bench.py --workload cfg3L --steps 50 --warmup 10 --no-e2e --no-cpu-baseline > $O/b3.json 2>$O/b3.err
python bench.py --workload cfg1 --steps 200 --warmup 20 --no-e2e --no-cpu-baseline > $O/b1.json 2>$O/b1.err
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/b4.json 2>$O/b4.err
for f in b3 b1 b4; do python -c "
import json;d=json.load(open('$O/$f.json'));print('$f', 'ms/step', d['ms_per_step'], 'value', d['value'], 'clk', d['clocks'].get('sm_mhz'), 'td3', d.get('td3',{}).get('ms_per_step'))"; done
