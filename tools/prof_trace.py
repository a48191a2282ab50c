"""Minimal driver for ncu captures of the trace kernel: build one format, trace the frame a few
times. Usage: python tools/prof_trace.py [--config cfg4] [--format SIG] [--restart] [--reps N]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench
import inputs
from paper_2410_14128_b200 import vf

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--format", default=None)
ap.add_argument("--restart", action="store_true")
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--counters", action="store_true")
ap.add_argument("--align", action="store_true", help="build with VF_BUILD_ALIGN_NODES")
ap.add_argument("--schedule", action="store_true", help="VF_TRACE_SCHEDULE launches (launch 2+ are ordered)")
ap.add_argument("--regroup", action="store_true", help="+ VF_TRACE_REGROUP (rays regrouped into warps)")
a = ap.parse_args()
vname, _, deffmt, _ = bench.CONFIGS[a.config]
vol = bench.make_volume(vname)
keys, rgba = inputs.voxels_device(vol)
h = vf.build((keys, rgba, inputs.dims_of(vol)), a.format or deffmt,
             flags=vf.VF_BUILD_DEFAULT | (vf.VF_BUILD_ALIGN_NODES if a.align else 0))
del keys, rgba
rays_np, _ = bench.make_rays(a.config)
rays = torch.from_numpy(rays_np).cuda()
hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
if a.counters:
    c = h.counters(rays, hits, restart=a.restart)
    n = c["rays"]
    print({k: round(v / n, 4) for k, v in c.items()})
for _ in range(a.reps):
    h.trace(rays, hits, restart=a.restart, schedule="regroup" if a.regroup else a.schedule)
torch.cuda.synchronize()
print(h.signature, h.stats()["bytes_used"])
