#!/bin/bash
# z-pass validation + variant sweep (values only; not bench lines)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2"
run() { echo "== $1"; shift; env "$@" timeout 300 $B > gpurun_out/sw.log 2>&1; python - <<'P'
import json
for l in open('gpurun_out/sw.log'):
    if l.startswith('{'):
        d = json.loads(l); print(' value %.1f frac %.3f iters %.1f' % (d['value'], d['roofline']['frac'], d['mean_iters_per_solve']))
        break
else:
    print(open('gpurun_out/sw.log').read()[-1500:])
P
}
run "z default (A: TY4 2/SM)" X=1
run "z minb1 (B: TY8 768)" DOT_COCG_MINB=1
run "z minb1 TY4 512" DOT_COCG_MINB=1 DOT_COCG_TY=4
run "z A PD3" DOT_COCG_PREFETCH=3
run "z B PD3" DOT_COCG_MINB=1 DOT_COCG_PREFETCH=3
run "z A PD1" DOT_COCG_PREFETCH=1
run "ring" DOT_COCG_KERNEL=ring
