"""Turn gpurun_out/ artefacts of tools/gpu_round.sh into the tracked profiles/ summaries.

  python tools/make_profiles.py r01
writes profiles/<tag>_launches.csv (raw ncu launch list), <tag>_launches_summary.txt
(per-kernel share of the step), <tag>_ncu_<kernel>.txt (ncu --set full key metrics),
cg_pass_traffic_<config>.json (DRAM traffic per launch of the CG pass vs its algorithmic
bytes, per captured grid; read by bench.py for that config) and <tag>_bench.jsonl (the bench line)."""
import collections, csv, json, os, shutil, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
G, P = "gpurun_out", "profiles"
os.makedirs(P, exist_ok=True)

# ---- launch list
rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("dot::<unnamed>::", "")
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
T = sum(tot.values())
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches.csv"))
with open(os.path.join(P, f"{tag}_launches_summary.txt"), "w") as fo:
    fo.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
    fo.write("# command: python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e (setup + 3 warm-up + 1 timed step)\n")
    fo.write(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        fo.write(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e6:10.2f} {v / T:7.4f}\n")
print(open(os.path.join(P, f"{tag}_launches_summary.txt")).read())

# ---- ncu --set full summaries
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]
traffic = {}
CAPTURES = (("prof_pass", "cg_pass", "full64", 64 ** 3), ("prof_contract", "contract", None, 0),
            ("prof_pass128", "cg_pass_all128", "all128", 128 ** 3), ("prof_pass96", "cg_pass_opt96", "opt96", 96 ** 3))
for rep, name, cfgname, npts in CAPTURES:
    path = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hh, units = r[0], r[1]
    lines = []
    for row in r[2:]:
        v = dict(zip(hh, row))
        lines.append(f"kernel {v.get('Kernel Name')}  grid {v.get('Grid Size')}  block {v.get('Block Size')}")
        for k in KEYS:
            if k in v:
                lines.append(f"  {k} = {v[k]} {units[hh.index(k)]}")
        st = sorted(((float(v[k]), k) for k in hh if k.startswith("smsp__average_warps_issue_stalled")
                     and k.endswith("per_issue_active.ratio") and v[k] not in ("", "n/a")), reverse=True)
        for val, k in st[:8]:
            lines.append(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} = {val:.3f}")
        if cfgname and cfgname not in traffic:
            gx, gy = [int(t) for t in v["Grid Size"].strip("()").split(",")[:2]]
            rd = float(v["dram__bytes_read.sum"]); wr = float(v["dram__bytes_write.sum"])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale[units[hh.index("dram__bytes_read.sum")]]
            wr *= scale[units[hh.index("dram__bytes_write.sum")]]
            n = round(npts ** (1 / 3))
            t = {"config": cfgname, "launch_pairs": gy, "grid": [gx, gy], "dram_bytes": rd + wr,
                 "algorithmic_bytes_if_all_active": 64.0 * npts * gy,
                 "note": (f"ncu --set full capture of one cg_pass_kernel launch ({gy} seed pairs, {n}^3): dram "
                          f"read+write per launch vs 32 B/point/seed algorithmic")}
            t["ratio"] = t["dram_bytes"] / t["algorithmic_bytes_if_all_active"]
            traffic[cfgname] = t
    with open(os.path.join(P, f"{tag}_ncu_{name}.txt"), "w") as fo:
        fo.write(f"# ncu --set full --clock-control none --import-source on ({rep}.ncu-rep), bench.py --profile\n")
        fo.write("\n".join(lines) + "\n")
    print("\n".join(lines))
for cfgname, t in traffic.items():
    json.dump(t, open(os.path.join(P, f"cg_pass_traffic_{cfgname}.json"), "w"), indent=1)
    print(t)
if os.path.exists(os.path.join(G, "sass_mix.txt")):
    shutil.copy(os.path.join(G, "sass_mix.txt"), os.path.join(P, f"{tag}_ncu_cg_pass_sass_mix.txt"))
bl = [l for l in open(os.path.join(G, "bench.log")) if l.startswith("{")]
if bl:
    open(os.path.join(P, f"{tag}_bench.jsonl"), "w").write(bl[-1])
