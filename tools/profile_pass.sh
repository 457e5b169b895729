#!/bin/bash
# one --set full capture of the COCG pass kernel (after a plain run of the same command)
CMD="python bench.py --profile --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cocg_pass_kernel -s 40 -c 1 -o gpurun_out/prof_pass $CMD > gpurun_out/ncu_full.log 2>&1
