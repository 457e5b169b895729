#!/bin/bash
# bench lines of the non-default rows (configs[1] sketch32, configs[3] opt96)
mkdir -p gpurun_out
for c in sketch32 opt96; do
  timeout 1200 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -c 2500 gpurun_out/bench_$c.log; echo
done
