# 1-pair (2 real seeds) solves at 96^3 -- the subspace iteration's real batches: pass efficiency
# over z-chunk counts, and the ncu kernel durations vs the event-timed pass time
mkdir -p gpurun_out
for zc in 0 4 6 8 10 12 16 24; do
  DOT_CG_ZCHUNKS=$zc timeout 600 python tools/pass_bench.py opt96 2 3 2>&1 | tail -1 | sed "s/^/zc=$zc /"
done
for xs in 1; do
  DOT_CG_XS=$xs timeout 600 python tools/pass_bench.py opt96 2 3 2>&1 | tail -1 | sed "s/^/xs=$xs /"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1pair.csv python tools/pass_bench.py opt96 2 1 > gpurun_out/ncu_1pair.log 2>&1; echo "ncu rc=$?"
python - <<'P'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_1pair.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum": continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")); cnt[name] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
    print(f"{k[:70]:70s} {cnt[k]:7d} {v / 1e6:9.2f} ms  {v / 1e3 / cnt[k]:8.2f} us/launch")
P
