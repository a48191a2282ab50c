"""Per-CUDA-source-line summary of `ncu --page source --csv --print-source cuda,sass`:
share of warp-stall samples, warp instructions and thread instructions per unit (e.g. per ray)."""
import csv
import sys

path = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
rows = list(csv.reader(open(path)))


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


hdr = None
lines = []
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        lines.append((fname, int(r[0]), r[1].strip()[:95], num(r[4]), num(r[7]), num(r[8])))
ts = sum(l[3] for l in lines) or 1
ti = sum(l[4] for l in lines)
tt = sum(l[5] for l in lines)
print(f"samples {ts:.0f}  warp-inst/unit {ti / units:.1f}  thread-inst/unit {tt / units:.1f}  SIMT {tt / max(ti, 1):.2f}")
print("file:line | %samples | warp-inst/unit | thread-inst/unit | avg thr | source")
lines.sort(key=lambda l: -l[3])
for l in lines[:top]:
    print(f"{l[0][:10]}:{l[1]:<4d} {l[3] / ts:6.1%} {l[4] / units:7.2f} {l[5] / units:8.2f} {l[5] / max(l[4], 1):5.1f}  {l[2]}")
