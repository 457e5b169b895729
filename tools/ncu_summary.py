"""Summarise an ncu report (raw page): time, DRAM traffic, stalls, pipes."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units = r[0], r[1]
for row in r[2:]:
    v = dict(zip(h, row))
    print(v.get("Kernel Name"), v.get("Grid Size"), v.get("Block Size"))
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
              "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
        if k in v:
            print(f"  {k} = {v[k]} {units[h.index(k)]}")
    st = sorted(((float(v[k]), k) for k in h if k.startswith("smsp__average_warps_issue_stalled")
                 and k.endswith("per_issue_active.ratio") and v[k] not in ("", "n/a")), reverse=True)
    for val, k in st[:8]:
        print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} = {val:.3f}")
