#!/bin/bash
# ncu --set full of one mid-solve CG pass launch of the default bench step (run under gpurun).
mkdir -p gpurun_out
PCMD="python bench.py --profile --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
timeout 600 $PCMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s ${SKIP:-420} -c 1 \
    -o gpurun_out/prof_pass $PCMD > gpurun_out/ncu_pass.log 2>&1; echo "ncu pass rc=$?"
python tools/sass_mix.py gpurun_out/prof_pass.ncu-rep > gpurun_out/sass_mix.txt 2>&1
