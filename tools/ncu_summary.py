"""Summarise an ncu report: key raw metrics and the top stall sites."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h:60s} {vals[i]:>16s} {units[i]}")
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        v = float(vals[i] or 0)
        if v > 0:
            print(f"  {h[33:]:40s} {v:10.0f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = srows[1]
ci = {k: i for i, k in enumerate(h)}
lst = []
tot = 0
for r in srows[2:]:
    try:
        v = float(r[ci["Warp Stall Sampling (All Samples)"]])
    except Exception:
        continue
    tot += v
    lst.append((v, r[ci["Address"]][-5:], r[ci["Source"]]))
print("top stall sites (% of samples):")
for v, a, s in sorted(lst, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {100 * v / tot:5.1f}%  {a}  {s}")
