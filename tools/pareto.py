"""Pareto frontier (fig:figure_1/2: rendering performance vs storage size, lower
bytes and higher Mrays/s better) of a bench.py JSON line's format sweep, stack variant, plus the
restart-sv gain per format (fig:restart-sv). usage: python tools/pareto.py BENCH_JSON [SWEEP_JSON]"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
if len(sys.argv) > 2:  # bench.py --sweep --sweep-out FILE
    d["sweep"] = json.load(open(sys.argv[2]))["rows"]
rows = [r for r in d.get("sweep", []) if "mrays_s" in r]
stack = {r["format"]: r for r in rows if r["variant"] == "stack"}
restart = {r["format"]: r for r in rows if r["variant"] == "restart"}
pts = sorted(stack.values(), key=lambda r: (r["paper_bytes_per_voxel"], -r["mrays_s"]))
front, best = [], -1.0
for r in pts:  # ascending size: on the frontier iff faster than every smaller format
    if r["mrays_s"] > best:
        front.append(r["format"])
        best = r["mrays_s"]
print(f"### Pareto frontier — {d['config']['workload']} (stack; paper-layout bytes per non-empty voxel)\n")
print("| format | B/voxel | Mrays/s | on frontier | restart-sv speed-up |")
print("|---|---|---|---|---|")
for r in sorted(stack.values(), key=lambda r: r["paper_bytes_per_voxel"]):
    rs = restart.get(r["format"])
    gain = f"{rs['mrays_s'] / r['mrays_s']:.2f}x" if rs else "—"
    print(f"| {r['format']} | {r['paper_bytes_per_voxel']} | {r['mrays_s']} | {'**yes**' if r['format'] in front else ''} | {gain} |")
print(f"\nfrontier: {', '.join(front)}")
if any(r.get("mrays_s_scheduled") for r in stack.values()):  # the same with VF_TRACE_SCHEDULE
    front_s, best = [], -1.0
    for r in sorted(stack.values(), key=lambda r: (r["paper_bytes_per_voxel"], -(r.get("mrays_s_scheduled") or 0))):
        if (r.get("mrays_s_scheduled") or 0) > best:
            front_s.append(r["format"])
            best = r["mrays_s_scheduled"]
    print(f"\nwith VF_TRACE_SCHEDULE (Mrays/s scheduled): frontier: " + ", ".join(
        f"{f} ({stack[f]['mrays_s_scheduled']})" for f in front_s))
