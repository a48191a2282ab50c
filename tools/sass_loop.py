"""Static SASS proxy for A/B of trace-loop code variants (no GPU): finds the outermost loop of a
kernel (widest backward branch) and counts its instructions by opcode class.
python tools/sass_loop.py LIB [kernel-substring]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else "trace_kernelILj5ELb0ELb0E"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
ins, on = [], False
for line in out.splitlines():
    if "Function :" in line:
        on = pat in line
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, t in ins:
    m = re.search(r"BRA\s+(?:`\()?\.?L?_?x?_?(0x[0-9a-f]+|\d+)", t)
    if m:
        try:
            tgt = int(m.group(1), 16)
        except ValueError:
            continue
        if tgt < a and (best is None or a - tgt > best[1] - best[0]):
            best = (tgt, a)
lo, hi = best
body = [t for a, t in ins if lo <= a <= hi]
cls = Counter()
for t in body:
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    k = "MOV" if ("MOV" in op and not op.startswith("UMOV")) else op.split(".")[0]
    cls[k] += 1
print(f"loop {lo:#x}-{hi:#x}: {len(body)} instructions; " + ", ".join(f"{k} {v}" for k, v in cls.most_common(14)))
