"""Per-reason stall samples by opcode of an ncu report (kernel source page)."""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
src = h.index("Source")
sc = {c: i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c}
tot = {}
for reason, i in sc.items():
    byop = collections.Counter()
    for r in data:
        if len(r) > i and r[i].isdigit():
            t = r[src].strip().split()
            op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
            byop[op] += int(r[i])
    tot[reason] = byop
T = sum(sum(b.values()) for b in tot.values())
for reason, byop in sorted(tot.items(), key=lambda x: -sum(x[1].values()))[:8]:
    print(f"{reason:22s} {sum(byop.values()) / T:.3f}", byop.most_common(5))
