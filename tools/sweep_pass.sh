#!/bin/bash
# COCG pass tiling sweep on the bench workload (values only; not a bench line)
for cfg in "225 512" "110 256" "112 256" "225 256"; do
  set -- $cfg
  DOT_COCG_SMEM_KB=$1 DOT_COCG_THREADS=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > gpurun_out/sweep_$1_$2.log 2>&1
done
