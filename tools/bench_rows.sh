#!/bin/bash
# bench lines of the non-default rows (configs[1] sketch32, configs[3] opt96)
mkdir -p gpurun_out
for c in sketch32 opt96; do
  K=3; [ $c = sketch32 ] && K=30     # sketch32 steps are ~10 ms: time more of them
  timeout 1200 python bench.py --config $c --no-cpu-baseline --steps $K --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -c 2500 gpurun_out/bench_$c.log; echo
done
