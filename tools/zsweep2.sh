#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2"
run() { echo "== $1"; shift; env "$@" timeout 300 $B > gpurun_out/sw.log 2>&1; python - <<'P'
import json
for l in open('gpurun_out/sw.log'):
    if l.startswith('{'):
        d = json.loads(l); print(' value %.1f frac %.3f' % (d['value'], d['roofline']['frac']))
        break
else:
    print(open('gpurun_out/sw.log').read()[-1500:])
P
}
run "ring cs1" DOT_COCG_KERNEL=ring
run "ring cs2" DOT_COCG_KERNEL=ring DOT_COCG_CLUSTER=2
run "ring cs4" DOT_COCG_KERNEL=ring DOT_COCG_CLUSTER=4
run "zB cs2" DOT_COCG_MINB=1 DOT_COCG_CLUSTER=2
run "zB cs4" DOT_COCG_MINB=1 DOT_COCG_CLUSTER=4
run "zB cs8" DOT_COCG_MINB=1 DOT_COCG_CLUSTER=8
run "zA cs2" DOT_COCG_CLUSTER=2
run "zA cs4" DOT_COCG_CLUSTER=4
run "zA cs8" DOT_COCG_CLUSTER=8
run "zA1 TY4 minb1 cs8" DOT_COCG_MINB=1 DOT_COCG_TY=4 DOT_COCG_CLUSTER=8
