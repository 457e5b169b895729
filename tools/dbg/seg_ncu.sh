# ncu --set full of the segment GEMM under tools/seg_bench.py (CONFIGS, default full64), library variant $V
mkdir -p gpurun_out
V=${V:-}
LP=""; [ -n "$V" ] && LP="DOT_LIB_PATH=$PWD/paper_1706_05586_b200/lib/variants/$V.so"
for c in ${CONFIGS:-full64}; do
  env $LP timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_tma_gemm -s ${SKIP:-2} -c 1 \
      -o gpurun_out/prof_seg_${c}${V:+_$V} python tools/seg_bench.py $c > gpurun_out/ncu_seg_$c.log 2>&1; echo "ncu $c rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_seg_${c}${V:+_$V}.ncu-rep 2>&1 | head -40
done
