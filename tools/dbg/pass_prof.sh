# CG pass at one config / seed count: GB/s (pass_bench) + ncu --set full of one mid-solve launch
mkdir -p gpurun_out
C=${CONFIG:-all128}; N=${NCOLS:-512}
timeout 600 python tools/pass_bench.py $C $N 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s ${SKIP:-40} -c 1 \
    -o gpurun_out/prof_pass_${C}_$N python tools/pass_bench.py $C $N 1 > gpurun_out/ncu_pass_${C}.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_pass_${C}_$N.ncu-rep | head -40
python tools/dbg/stall_ops.py gpurun_out/prof_pass_${C}_$N.ncu-rep
