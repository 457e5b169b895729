# 128^3 pass: x split forced vs default, GB/s and one ncu capture of the split launch
for m in 0 2; do DOT_CG_XS=$m timeout 900 python tools/pass_bench.py all128 512 1 2>&1 | tail -1 | sed "s/^/xs=$m /"; done
DOT_CG_XS=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_pass_kernel -s 40 -c 1 -o gpurun_out/prof_pass128_xs2 python tools/pass_bench.py all128 512 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_pass128_xs2.ncu-rep | head -32
python tools/dbg/stall_ops.py gpurun_out/prof_pass128_xs2.ncu-rep
