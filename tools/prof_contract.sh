#!/bin/bash
# ncu --set full of the block-sparse Jacobian contraction of the default bench step (run under gpurun).
mkdir -p gpurun_out
PCMD="python bench.py --profile --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
timeout 600 $PCMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:seg_tma_gemm -c 1 \
    -o gpurun_out/prof_contract $PCMD > gpurun_out/ncu_contract.log 2>&1; echo "ncu contract rc=$?"
