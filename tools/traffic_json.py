"""Merge an ncu --csv dram-bytes pass over tools/sweep_trace.py into profiles/traffic.json.
usage: python tools/traffic_json.py NCU_CSV SWEEP_STDOUT"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
launch = {}
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    if "trace_kernel" not in d["Kernel Name"] and "trace_persistent" not in d["Kernel Name"]:
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
             "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}.get(unit, 1)
    launch.setdefault(int(d["ID"]), {})[d["Metric Name"]] = v * scale
launches = [l.split()[1:] for l in open(sys.argv[2]) if l.startswith("LAUNCH ")]
keys = [" ".join(x[:-1]) if x[-1].isdigit() else " ".join(x) for x in launches]
nrays = [int(x[-1]) if x[-1].isdigit() else None for x in launches]
ids = sorted(launch)
path = os.path.join(ROOT, "profiles", "traffic.json")
tj = json.load(open(path)) if os.path.exists(path) else {}
for key, i, nr in zip(keys, ids, nrays):
    m = launch[i]
    tj[key] = {"dram_bytes_per_launch": int(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)),
               "ncu_duration_ns": int(m.get("gpu__time_duration.sum", 0)),
               "warp_inst_per_launch": int(m.get("smsp__inst_executed.sum", 0)),
               "thread_inst_per_launch": int(m.get("smsp__thread_inst_executed.sum", 0)),
               "rays": nr,
               "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                         "smsp__inst_executed.sum,smsp__thread_inst_executed.sum "
                         "--clock-control none over tools/sweep_trace.py (cold cache, serialised)"}
json.dump(tj, open(path, "w"), indent=1, sort_keys=True)
print(f"{len(keys)} launches merged into {path}")
