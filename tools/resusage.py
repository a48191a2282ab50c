"""Registers / stack per trace kernel instantiation: python tools/resusage.py [libvf.so]"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2410_14128_b200/libvf.so"
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
name = None
for line in out.split("\n"):
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and name and "trace_" in name:
        k = re.search(r"trace_(kernel|persistent)ILj(\d+)ELb([01])ELb([01])", name)
        if not k:
            continue
        print(f"{k.group(1):10s} kinds={int(k.group(2)):2d} restart={k.group(3)} count={k.group(4)} "
              f"REG={m.group(1)} STACK={m.group(2)}")
