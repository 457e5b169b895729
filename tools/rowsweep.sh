#!/bin/bash
# sweep env settings on one bench config: rowsweep.sh CONFIG "ENV=.. ENV=.." ...
c=$1; shift
for v in "$@"; do
  env $v timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/rs.log 2>&1
  python - "$v" <<'P'
import json, sys
for l in open('gpurun_out/rs.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], ' value %.1f frac %.4f' % (d['value'], d['roofline']['frac'])); break
else:
    print(sys.argv[1], open('gpurun_out/rs.log').read()[-600:])
P
done
