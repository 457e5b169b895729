# x-split pass: parity with DOT_CG_XS=2 forced on the small-grid suite, then pass GB/s xs=1 vs default
mkdir -p gpurun_out
DOT_CG_XS=2 timeout 1200 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -4
for cfgn in ${ROWS:-"all128 512" "opt96 20" "opt96 60"}; do
  set -- $cfgn
  for m in 1 0; do
    DOT_CG_XS=$m timeout 900 python tools/pass_bench.py $1 $2 1 2>&1 | tail -1 | sed "s/^/xs=$m /"
  done
done
