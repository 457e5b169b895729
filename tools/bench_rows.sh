#!/bin/bash
# bench lines of the non-default rows (configs[1] sketch32, configs[3] opt96, configs[4] all128)
mkdir -p gpurun_out
for c in ${ROWS:-sketch32 opt96 all128}; do
  K=3; [ $c = sketch32 ] && K=30     # sketch32 steps are ~10 ms: time more of them
  [ $c = all128 ] && K=1
  timeout 1800 python bench.py --config $c --no-cpu-baseline --steps $K --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], round(d["value"],1), d["unit"], "ms/step", round(d["ms_per_step"],1), "pass frac", round(d["roofline"]["frac"],3), "J tflops", round(d["jacobian"]["achieved_tflops"],2), "e2e", d["e2e"] and round(d["e2e"]["value"],1))'
done
