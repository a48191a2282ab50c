"""Markdown summary of one `ncu --set full` capture from its exported pages (tools/gpu_pack.sh:
<base>_raw.csv, <base>_details.csv, <base>_source.csv.gz), for profiles/.
usage: python tools/summarize_ncu_csv.py BASE UNITS_PER_LAUNCH LABEL"""
import csv
import gzip
import sys
from collections import Counter

base, units, label = sys.argv[1], float(sys.argv[2]), sys.argv[3]
raw = list(csv.reader(open(base + "_raw.csv")))
R = {h: (v, u) for h, u, v in zip(raw[0], raw[1], raw[2])}
det = list(csv.reader(open(base + "_details.csv")))
D, kname = {}, ""
for r in det[1:]:
    d = dict(zip(det[0], r))
    kname = d.get("Kernel Name", kname)
    D[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def g(name):
    v = D.get(name) or R.get(name)
    return f"{v[0]} {v[1]}".strip() if v else "n/a"


def num(name):
    v = R.get(name) or D.get(name)
    try:
        return float(v[0].replace(",", "")) * SCALE.get(v[1], 1)
    except Exception:
        return float("nan")


print(f"# ncu summary — {label}\n\nkernel: `{kname}`\n\n| metric | value |\n|---|---|")
for m in ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "Compute (SM) Throughput",
          "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
          "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
          "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
          "No Eligible", "Branch Efficiency", "Executed Instructions", "Grid Size", "Block Size"]:
    print(f"| {m} | {g(m)} |")
for m in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
          "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sector_hit_rate.pct",
          "l1tex__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread"]:
    print(f"| {m} | {g(m)} |")
dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
print(f"\nPer unit ({units:.0f} units per launch): DRAM {dram / units:.1f} B, L2 {num('lts__t_bytes.sum') / units:.1f} B, "
      f"L1 {num('l1tex__t_bytes.sum') / units:.1f} B, "
      f"{num('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum') / units:.1f} global-load sectors, "
      f"{num('smsp__inst_executed.sum') / units:.1f} warp instructions\n")
rows = list(csv.reader(gzip.open(base + "_source.csv.gz", "rt")))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall = Counter()
tot = 0
for r in rows[2:]:
    for h in hdr:
        if h.startswith("stall_") and "(Not Issued)" not in h:
            try:
                stall[h] += int(r[ix[h]])
            except ValueError:
                pass
    tot += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("## warp-state samples (all samples)\n\n| reason | share |\n|---|---|")
for k, v in stall.most_common(10):
    print(f"| {k} | {100 * v / max(tot, 1):.1f} % |")
