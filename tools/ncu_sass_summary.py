"""Summarise an `ncu --page source --csv` SASS dump: stall-reason totals and the hottest
instructions (by warp-stall samples and by executed instructions)."""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for d in data:
    for c in stall_cols:
        tot[c] += num(d[c])
S = sum(tot.values())
print("stall reasons (share of all samples):")
for k, v in tot.most_common(12):
    print(f"  {k:28s} {v / S:6.1%}")
ie = sum(num(d["Instructions Executed"]) for d in data)
te = sum(num(d["Thread Instructions Executed"]) for d in data)
print(f"instructions executed {ie:.4g}, thread instr {te:.4g}, avg threads/instr {te / max(ie, 1):.2f}")
print(f"\ntop {top} by samples: addr | samples | inst exec | avg thr | source")
data.sort(key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))
for d in data[:top]:
    print(f"  {d['Address']:>6} {num(d['Warp Stall Sampling (All Samples)']):7.0f} {num(d['Instructions Executed']):10.0f} "
          f"{num(d['Avg. Threads Executed']):5.1f}  {d['Source'][:90]}")
