#!/bin/bash
# A/B of library variants / env knobs on the default bench (values only, not bench lines).
#   VARIANTS="label1:ENV=VAL+ENV2=VAL label2:" bash tools/ab_bench.sh [bench args]
for v in ${VARIANTS:-"default:"}; do
  label=${v%%:*}; envs=$(echo "${v#*:}" | tr "+" " ")
  out=$(env $envs python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1)
  echo "$label $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],2), round(d["roofline"]["frac"],4))' 2>&1)"
done
