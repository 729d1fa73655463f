"""Key metrics of the first kernel in an ncu report: python scripts/ncu_summary.py rep.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u, v = r[0], r[1], r[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "l1tex__t_sector_hit_rate.pct", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]} {u[h.index(k)]}")
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            if float(v[i]) >= 0.1:
                print(f"{k:70s} {v[i]}")
        except ValueError:
            pass
for i, k in enumerate(h):
    if k.startswith("sm__inst_executed_pipe_") and k.endswith("avg.pct_of_peak_sustained_active"):
        try:
            if float(v[i]) >= 5:
                print(f"{k:70s} {v[i]}")
        except ValueError:
            pass
