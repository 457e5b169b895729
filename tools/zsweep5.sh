#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -5
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2"
run() { echo "== $1"; shift; env "$@" timeout 300 $B > gpurun_out/sw.log 2>&1; python - <<'P'
import json
for l in open('gpurun_out/sw.log'):
    if l.startswith('{'):
        d = json.loads(l); print(' value %.1f frac %.3f iters %.3f misfit %.10e' % (d['value'], d['roofline']['frac'], d['mean_iters_per_solve'], d['misfit']))
        break
else:
    print(open('gpurun_out/sw.log').read()[-1500:])
P
}
for v in "$@"; do run "$v" $v; done
