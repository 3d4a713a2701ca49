"""Key metrics of an ncu report (first kernel): python tools/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
d = {a: (c, b) for a, b, c in zip(h, u, v)}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
for k in keys:
    if k in d:
        print(f"{k:60s} {d[k][0]:>18s} {d[k][1]}")
st = sorted([(float(c.replace(',', '')), a) for a, (c, b) in d.items()
             if a.startswith("smsp__pcsamp_warps_issue_stalled") and not a.endswith("not_issued")
             and c.replace(',', '').replace('.', '').isdigit()], reverse=True)[:8]
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{a.replace('smsp__pcsamp_warps_issue_stalled_', '')}={x/tot:.0%}" for x, a in st))
