"""Instruction mix and stall attribution of one kernel from an ncu --set full report.

  python tools/sass_mix.py REPORT.ncu-rep > profiles/<tag>_ncu_<kernel>_sass_mix.txt
Reads `ncu -i REPORT --page source --csv --print-source sass`, sums executed warp
instructions and warp-stall samples per opcode, and lists the most-stalled
instructions with their dominant stall reason."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kernel = rows[0][1] if rows and len(rows[0]) > 1 else "?"
h, data = rows[1], rows[2:]
ie, src, samp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
byop, sampop, tot, tots = collections.Counter(), collections.Counter(), 0, 0
byreason = collections.Counter()
hot = []
for r in data:
    if len(r) <= max(ie, samp) or not r[ie].isdigit():
        continue
    n, s = int(r[ie]), int(r[samp]) if r[samp].isdigit() else 0
    toks = r[src].strip().split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
    byop[op] += n
    sampop[op] += s
    tot += n
    tots += s
    reasons = [(int(r[i]) if r[i].isdigit() else 0, c) for i, c in stall_cols]
    for v, c in reasons:
        byreason[c] += v
    hot.append((s, r[src].strip(), max(reasons)[1] if reasons else "-"))
print(f"# {kernel}")
print(f"# {rep}: {tot} warp instructions executed, {tots} warp-stall samples")
print(f"{'opcode':10s} {'instr share':>11s} {'stall share':>11s}")
for op, n in byop.most_common(20):
    print(f"{op:10s} {n / tot:11.3f} {sampop[op] / max(tots, 1):11.3f}")
print("\n# stall reasons (share of samples)")
rs = sum(byreason.values())
for c, v in byreason.most_common(8):
    print(f"{c:32s} {v / max(rs, 1):.3f}")
print("\n# most-stalled instructions (samples, dominant reason)")
for s, t, c in sorted(hot, reverse=True)[:10]:
    print(f"{s:7d}  {c:24s} {t[:70]}")
