"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total
device time and share (cold-cache, serialised launches: compare SHARES, not absolutes)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].isdigit()]
agg = defaultdict(lambda: [0, 0.0])
for d in data:
    agg[d["Kernel Name"].split("(")[0][:90]][0] += 1
    agg[d["Kernel Name"].split("(")[0][:90]][1] += float(d["Metric Value"].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print("kernel,launches,total_us,mean_us,share")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"\"{k}\",{v[0]},{v[1] / 1e3:.1f},{v[1] / 1e3 / v[0]:.1f},{v[1] / tot:.4f}")
