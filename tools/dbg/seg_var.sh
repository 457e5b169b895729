# segment GEMM: library variants (DOT_LIB_PATH) on tools/seg_bench.py
for v in "$@"; do
  echo "== $v"; DOT_LIB_PATH=$PWD/paper_1706_05586_b200/lib/variants/$v.so timeout 600 python tools/seg_bench.py ${CONFIGS:-full64}
done
