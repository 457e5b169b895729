# Two-stream pass groups (half batches on two streams fill each other's wave tails) and the
# opt96 field-cache reuse: parity first, then A/B against DOT_CG_NOSPLIT=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x 2>&1 | tail -2 | sed "s/^/parity: /"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "opt96 or certified" 2>&1 | tail -2 | sed "s/^/fullsize: /"
for v in 0 1; do
  DOT_CG_NOSPLIT=$( [ $v = 1 ] && echo 1 ) timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/split_bench_$v.log 2>&1
  tail -1 gpurun_out/split_bench_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("nosplit='$v'", round(d["value"],1), "pass", round(d["roofline"]["frac"],4), "ms", round(d["ms_per_step"],2), "J", d["jacobian"]["gemm"], d["clocks"]["sm_mhz"])'
done
for v in 0 1; do
  if [ $v = 1 ]; then export DOT_CG_NOSPLIT=1; else unset DOT_CG_NOSPLIT; fi
  timeout 900 python tools/pass_bench.py all128 512 1 2>&1 | tail -1 | sed "s/^/nosplit=$v /"
  timeout 900 python tools/pass_bench.py opt96 60 1 2>&1 | tail -1 | sed "s/^/nosplit=$v /"
done
unset DOT_CG_NOSPLIT
timeout 900 python bench.py --config opt96 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/split_opt96.log 2>&1
tail -1 gpurun_out/split_opt96.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("opt96", round(d["value"],1), "ms", round(d["ms_per_step"],1), "solves", d["config"]["solves_per_step"], "pass", round(d["roofline"]["frac"],4))'
