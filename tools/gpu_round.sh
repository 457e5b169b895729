#!/bin/bash
# One GPU round: smoke, GPU parity suite, default bench line, ncu launch list of a
# short bench, ncu --set full of the CG pass and the Jacobian contraction.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log
if [ "${SKIP_NCU:-0}" = "1" ]; then exit 0; fi
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
PCMD="python bench.py --profile --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 $PCMD > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s 420 -c 1 -o gpurun_out/prof_pass $PCMD > gpurun_out/ncu_pass.log 2>&1; echo "ncu pass rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_seg -c 1 -o gpurun_out/prof_contract $PCMD > gpurun_out/ncu_contract.log 2>&1; echo "ncu contract rc=$?"
python tools/sass_mix.py gpurun_out/prof_pass.ncu-rep > gpurun_out/sass_mix.txt 2>&1
ls -la gpurun_out
