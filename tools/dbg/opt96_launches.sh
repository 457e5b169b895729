# kernel-time breakdown of one opt96 bench step (ncu launch list) vs the step's wall time
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_opt96.csv python bench.py --config opt96 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/opt96_ncu.log 2>&1; echo "rc=$?"
python - <<'P'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_opt96.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum": continue
    name = r[ki].split("(")[0].replace("void ", "").replace("dot::<unnamed>::", "")
    tot[name] += float(r[vi].replace(",", "")); cnt[name] += 1
T = sum(tot.values())
print("total kernel ms (setup + 1 warm + 1 timed step):", T / 1e6)
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
    print(f"{k[:62]:62s} {cnt[k]:7d} {v / 1e6:9.2f} {v / T:6.3f}")
P
