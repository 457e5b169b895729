#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run, then the launch list, then one
# --set full capture of the COCG pass kernel.  Run under gpurun from the repo root.
set -e
CMD="python bench.py --profile --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cocg_pass_kernel -s 40 -c 1 -o gpurun_out/prof_pass $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 0 -c 1 -o gpurun_out/prof_contract $CMD > gpurun_out/ncu_full2.log 2>&1
