#!/bin/bash
# lean bench sweep (no tests): lsweep.sh "ENV=.." ...
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2"
for v in "$@"; do
  env $v timeout 300 $B > gpurun_out/ls.log 2>&1
  python - "$v" <<'P'
import json, sys
for l in open('gpurun_out/ls.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], ' value %.1f frac %.4f iters %.3f' % (d['value'], d['roofline']['frac'], d['mean_iters_per_solve'])); break
else:
    print(sys.argv[1], open('gpurun_out/ls.log').read()[-600:])
P
done
