"""A/B timing of libvf.so variants on the same box: python tools/ab.py LIB1,LIB2 CFG:FORMAT ...
Alternates variants (A B A B) in fresh processes; prints median Mrays/s (stack and restart)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, statistics, torch, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import bench, inputs
from paper_2410_14128_b200 import vf
out = []
cache = {}
for spec in sys.argv[1:]:
    cfg, fmt = spec.split(":", 1)
    vname, _, deffmt, _ = bench.CONFIGS[cfg]
    if cfg not in cache:
        vol = bench.make_volume(vname)
        cache.clear()
        cache[cfg] = (vol, inputs.voxels_device(vol), bench.make_rays(cfg)[0])
    vol, (k, c), rays_np = cache[cfg]
    h = vf.build((k, c, inputs.dims_of(vol)), fmt or deffmt)
    rays = torch.from_numpy(rays_np).cuda()
    hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
    flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
    res = []
    for restart in (False, True):
        for _ in range(3): h.trace(rays, hits, restart=restart)
        ms = []
        for i in range(15):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); h.trace(rays, hits, restart=restart); b.record()
            torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
        res.append(rays.shape[0] / statistics.median(ms) / 1e3)
    out.append(f"{spec}: stack {res[0]:.0f} restart {res[1]:.0f}")
    h.close()
print(" | ".join(out))
'''
libs = sys.argv[1].split(",")
specs = sys.argv[2:]
for rep in range(2):
    for lib in libs:
        env = dict(os.environ, ROOT=ROOT, VF_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", code, *specs], env=env, capture_output=True, text=True)
        print(f"[{rep}] {lib}: {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
