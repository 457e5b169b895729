#!/bin/bash
mkdir -p gpurun_out
export DOT_COCG_MINB=1
PCMD="python bench.py --profile --no-cpu-baseline --no-e2e"
timeout 600 $PCMD > gpurun_out/plainz.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cocg_zpass -s 40 -c 1 -o gpurun_out/prof_zB $PCMD > gpurun_out/ncu_zB.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_zB.log
