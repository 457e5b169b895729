#!/bin/bash
mkdir -p gpurun_out
PCMD="python bench.py --profile --no-cpu-baseline --no-e2e"
timeout 600 $PCMD > gpurun_out/plainz.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cocg_zpass -s 40 -c 1 -o gpurun_out/prof_zD $PCMD > gpurun_out/ncu_z.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_z.log
