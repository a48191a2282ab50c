"""Write a markdown summary of one `ncu --set full` capture (.ncu-rep) for profiles/.
usage: python tools/summarize_ncu.py REP.ncu-rep UNITS_PER_LAUNCH LABEL > profiles/NAME.md"""
import csv
import io
import subprocess
import sys

rep, units, label = sys.argv[1], float(sys.argv[2]), sys.argv[3]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


details = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
hdr = details[0]
D = {}
kname = ""
for r in details[1:]:
    d = dict(zip(hdr, r))
    kname = d.get("Kernel Name", kname)
    D[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
R = {h: (v, u) for h, u, v in zip(raw[0], raw[1], raw[2])}


def g(name):
    v = D.get(name) or R.get(name)
    return f"{v[0]} {v[1]}".strip() if v else "n/a"


def f(name):
    try:
        return float((R.get(name) or D.get(name))[0].replace(",", ""))
    except Exception:
        return float("nan")


rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
unit_r = (R.get("dram__bytes_read.sum") or ("", ""))[1]
unit_w = (R.get("dram__bytes_write.sum") or ("", ""))[1]
dram = rd * SCALE.get(unit_r, 1) + wr * SCALE.get(unit_w, 1)  # (read and write may differ in unit)
print(f"# ncu summary — {label}\n")
print(f"kernel: `{kname}`\n")
print("| metric | value |\n|---|---|")
for m in ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "Compute (SM) Throughput",
          "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
          "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
          "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
          "No Eligible", "Branch Efficiency", "Executed Instructions", "Grid Size", "Block Size"]:
    print(f"| {m} | {g(m)} |")
for m in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
          "lts__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
    print(f"| {m} | {g(m)} |")
print(f"\nDRAM traffic per launch (read+write): {dram:.4g} B = {dram / units:.2f} B per unit ({units:.0f} units)\n")
src = ncu("--page", "source", "--csv", "--print-source", "cuda,sass")
open("/tmp/_src.csv", "w").write(src)
out = subprocess.run([sys.executable, __file__.replace("summarize_ncu.py", "ncu_line_summary.py"), "/tmp/_src.csv",
                      str(units), "25"], capture_output=True, text=True).stdout
print("## hottest source lines (warp-stall samples; instructions per unit)\n\n```\n" + out + "```")
sass = ncu("--page", "source", "--csv")
open("/tmp/_sass.csv", "w").write(sass)
out = subprocess.run([sys.executable, __file__.replace("summarize_ncu.py", "ncu_sass_summary.py"), "/tmp/_sass.csv",
                      "0"], capture_output=True, text=True).stdout
print("## stall reasons\n\n```\n" + out + "```")
