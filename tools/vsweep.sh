#!/bin/bash
# bench the library variants in paper_1706_05586_b200/lib/variants (values only)
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2"
for rep in 1 2; do
for v in "$@"; do
  DOT_LIB_PATH=$PWD/paper_1706_05586_b200/lib/variants/$v.so timeout 300 $B > gpurun_out/vs.log 2>&1
  python - "$v" <<'P'
import json, sys
for l in open('gpurun_out/vs.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], ' value %.1f frac %.4f iters %.3f' % (d['value'], d['roofline']['frac'], d['mean_iters_per_solve'])); break
else:
    print(sys.argv[1], open('gpurun_out/vs.log').read()[-800:])
P
done; done
