# A/B of the segment contraction kernels (values only): DOT_SEG_V1 (round-2a kernel) / default (pre-formed operand tiles)
mkdir -p gpurun_out
for v in ${VARIANTS:-v1 v4}; do
  unset DOT_SEG_V1
  [ $v = v1 ] && export DOT_SEG_V1=1
  echo "== $v"; timeout 600 python tools/seg_bench.py ${CONFIGS:-full64 all128}
done 2>&1 | tee gpurun_out/seg_ab.txt
