set -u
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
EVIDENCE_PART=bench bash tools/evidence.sh > gpurun_out/ev.log 2>&1; grep rc= gpurun_out/ev.log
SPIKERL_BENCH_COMM=1 python bench.py --workload cfg3L --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3L_comm.json 2> gpurun_out/bench_cfg3L_comm.err; echo "comm cfg3L rc=$?"
SPIKERL_BENCH_COMM=1 python bench.py --workload cfg1 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg1_comm.json 2> gpurun_out/bench_cfg1_comm.err; echo "comm cfg1 rc=$?"
