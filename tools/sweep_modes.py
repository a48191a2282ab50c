"""Time the trace kernel for one config/format under different launch modes / refill thresholds."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, statistics, torch, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import bench, inputs
from paper_2410_14128_b200 import vf
cfg, fmt = sys.argv[1], sys.argv[2]
vname, _, deffmt, _ = bench.CONFIGS[cfg]
vol = bench.make_volume(vname)
k, c = inputs.voxels_device(vol)
h = vf.build((k, c, inputs.dims_of(vol)), fmt or deffmt)
del k, c
rays_np, _ = bench.make_rays(cfg)
rays = torch.from_numpy(rays_np).cuda()
hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
res = {}
for restart in (False, True):
    for otpr in (False, True):
        for _ in range(3): h.trace(rays, hits, restart=restart, persistent=otpr)
        ms = []
        for i in range(10):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); h.trace(rays, hits, restart=restart, persistent=otpr); b.record()
            torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
        res[("restart" if restart else "stack", "persist" if otpr else "otpr")] = rays.shape[0] / statistics.median(ms) / 1e3
print(os.environ.get("VF_REFILL", "12"), h.signature, {f"{k[0]}/{k[1]}": round(v, 1) for k, v in res.items()})
'''
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
fmt = sys.argv[2] if len(sys.argv) > 2 else ""
blocks = sys.argv[4].split(",") if len(sys.argv) > 4 else ["128"]
for refill in sys.argv[3].split(",") if len(sys.argv) > 3 else ["12"]:
    for blk in blocks:
        env = dict(os.environ, ROOT=ROOT, VF_REFILL=refill, VF_BLOCK=blk)
        print("block", blk, end=" ", flush=True)
        subprocess.run([sys.executable, "-c", code, cfg, fmt], env=env)
