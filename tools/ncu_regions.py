"""Aggregate a `--print-source cuda,sass` ncu dump of trace.cu by code region: the regions are
delimited by the comment markers in csrc/trace.cu (root function / cell test / descent / step /
pop); lines above `struct Lane` are helpers (tplane, certified compares, locate, headers)."""
import csv
import re
import sys

src_path, csv_path, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
markers = [("// ---- root function", "start"), ("// -- test the current cell", "test"),
           ("// descend at event E", "descend"), ("// -- step: exact next event", "step"),
           ("// left the current node: pop", "pop"), ("__device__ __forceinline__ int4 hit_record", "kernel")]
lines = open(src_path).read().split("\n")
bounds = []
for i, l in enumerate(lines, 1):
    for m, name in markers:
        if m in l:
            bounds.append((i, name))
lane_start = next(i for i, l in enumerate(lines, 1) if l.startswith("struct Lane"))


def region(ln):
    if ln < lane_start:
        return "helpers"
    r = "lane-misc"
    for b, name in bounds:
        if ln >= b:
            r = name
    return r


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


agg = {}
fname = ""
for r in csv.reader(open(csv_path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0].isdigit():
        key = region(int(r[0])) if fname.endswith("trace.cu") else "other:" + fname.split("/")[-1]
        a = agg.setdefault(key, [0.0, 0.0, 0.0])
        a[0] += num(r[4])
        a[1] += num(r[7])
        a[2] += num(r[8])
ts = sum(v[0] for v in agg.values()) or 1
print("region        %samples  warp-inst/unit  thread-inst/unit  avg-threads")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:14s} {v[0] / ts:7.1%} {v[1] / units:12.1f} {v[2] / units:14.1f} {v[2] / max(v[1], 1):10.1f}")
