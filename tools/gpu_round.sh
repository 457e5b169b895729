#!/bin/bash
# One GPU round: smoke, GPU parity suite, default bench line, bench rows, ncu launch list of a
# short bench, ncu --set full of the CG pass (64^3 bench step, 128^3 and 96^3 pass_bench launches)
# and of the Jacobian segment GEMM.  SKIP_NCU=1: tests and bench lines only.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log
[ "${SKIP_ROWS:-0}" = "1" ] || bash tools/bench_rows.sh
if [ "${SKIP_NCU:-0}" = "1" ]; then exit 0; fi
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
PCMD="python bench.py --profile --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 $PCMD > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s 900 -c 1 -o gpurun_out/prof_pass $PCMD > gpurun_out/ncu_pass.log 2>&1; echo "ncu pass rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_tma_gemm -c 1 -o gpurun_out/prof_contract $PCMD > gpurun_out/ncu_contract.log 2>&1; echo "ncu contract rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s 40 -c 1 -o gpurun_out/prof_pass128 python tools/pass_bench.py all128 512 1 > gpurun_out/ncu_pass128.log 2>&1; echo "ncu pass128 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s 100 -c 1 -o gpurun_out/prof_pass96 python tools/pass_bench.py opt96 20 1 > gpurun_out/ncu_pass96.log 2>&1; echo "ncu pass96 rc=$?"
python tools/sass_mix.py gpurun_out/prof_pass.ncu-rep > gpurun_out/sass_mix.txt 2>&1
ls -la gpurun_out
