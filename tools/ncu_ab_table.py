"""Markdown table of ncu --metrics --csv captures (one launch each): python tools/ncu_ab_table.py LABEL=FILE ..."""
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9,
         "sector": 1, "Ksector": 1e3, "Msector": 1e6, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1, "msecond": 1e3,
         "nsecond": 1e-3}
cols, table = [], []
for arg in sys.argv[1:]:
    label, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    m = {}
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            m[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
        except ValueError:
            pass
    table.append((label, m))
    for k in m:
        if k not in cols:
            cols.append(k)
print("| metric | " + " | ".join(l for l, _ in table) + " |")
print("|---|" + "---|" * len(table))
for c in cols:
    print(f"| {c} | " + " | ".join(f"{m.get(c, float('nan')):.4g}" for _, m in table) + " |")
