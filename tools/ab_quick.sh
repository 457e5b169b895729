#!/bin/bash
# quick check of a pass-kernel change: GPU parity suite, pass throughput per batch size, bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
for rep in 1 2; do
  for spec in "sketch32 8 20" "sketch32 16 20" "opt96 2 3" "opt96 20 2" "full64 64 2" "full64 512 1" "all128 64 1"; do
    timeout 600 python tools/pass_bench.py $spec 2>&1 | tail -1
  done
done
for c in sketch32 opt96 full64; do
  K=3; [ $c = sketch32 ] && K=30
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps $K --warmup 3 > gpurun_out/bench_quick_$c.log 2>&1
  tail -1 gpurun_out/bench_quick_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], round(d["value"],1), "ms/step", round(d["ms_per_step"],2), "pass frac", round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])'
done
