# launch times of the contraction kernels in tools/seg_bench.py (CONFIG) + ncu --set full of one GEMM launch
mkdir -p gpurun_out
C=${CONFIG:-full64}
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"seg_" --csv python tools/seg_bench.py $C > gpurun_out/seg_launch_$C.csv 2>/dev/null; echo "launch rc=$?"
python - "$C" <<'P'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/seg_launch_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; data = rows[1:]
k, m, v = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in data:
    agg[(r[k][:40], r[m])].append(float(r[v].replace(",", "")))
for key, vals in sorted(agg.items()):
    print(key, len(vals), "mean %.4g" % (sum(vals) / len(vals)))
P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_tma_gemm -s ${SKIP:-3} -c 1 -o gpurun_out/prof_tma_$C python tools/seg_bench.py $C > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_tma_$C.ncu-rep | head -32
python tools/dbg/stall_ops.py gpurun_out/prof_tma_$C.ncu-rep
