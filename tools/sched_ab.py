"""A/B of VF_TRACE_SCHEDULE (longest-first block order from the previous launch over the same ray
array) on the configs' headline formats, same process, L2 flushed before every timed launch:
  natural  index order (the default launch)
  sched    order from the previous frame of the same camera
  moved-X  order from the previous frame of a camera moved by X of the eye-target distance (the
           previous frame's rays are copied into the buffer and traced, then this frame's rays)
Hits must be bit-identical in every mode.
Usage: python tools/sched_ab.py cfg4 cfg2 cfg5 [--restart]"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench
import inputs
from inputs import rays as R
from paper_2410_14128_b200 import vf

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--restart", action="store_true")
ap.add_argument("--reps", type=int, default=15)
a = ap.parse_args()

sys.path.insert(0, os.path.join(ROOT, "tools"))
from sched_common import CAM, moved_rays  # noqa: E402


flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
for cfg in a.configs:
    vname, _, fmt, _ = bench.CONFIGS[cfg]
    vol = bench.make_volume(vname)
    k, c = inputs.voxels_device(vol)
    h = vf.build((k, c, inputs.dims_of(vol)), fmt)
    del k, c
    rays_np = bench.make_rays(cfg)[0]
    rays = torch.from_numpy(rays_np).cuda()
    prev = {f: torch.from_numpy(moved_rays(CAM[cfg], f)).cuda() for f in (0.005, 0.05)}
    path = [torch.from_numpy(moved_rays(CAM[cfg], 0.001 * j)).cuda() for j in range(a.reps + 3)]
    n = rays.shape[0]
    buf = torch.empty_like(rays)
    hits = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    ref = h.trace(rays).clone()
    res = {}
    for rep in range(2):
        for mode in ("natural", "sched", "regroup", "moved-0.005", "moved-0.005-regroup", "path-sched",
                     "path-regroup"):
            ms = []
            for i in range(a.reps + 3):
                sm = "regroup" if mode.endswith("regroup") else mode != "natural"
                if mode.startswith("path"):  # a moving camera: frame i of a path of 0.1 % steps
                    buf.copy_(path[i % len(path)])
                elif mode.startswith("moved"):
                    buf.copy_(prev[float(mode.split("-")[1])])
                    h.trace(buf, hits, restart=a.restart, schedule=sm)
                    buf.copy_(rays)
                else:
                    buf.copy_(rays)
                flush.fill_(i)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                h.trace(buf, hits, restart=a.restart, schedule=sm)
                e1.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ms.append(e0.elapsed_time(e1))
                if not mode.startswith("path"):
                    assert torch.equal(hits, ref), f"{cfg} {mode}: hits differ"
            res.setdefault(mode, []).append(statistics.median(ms))
    base = min(res["natural"])
    print(f"{cfg} {h.signature} {'restart' if a.restart else 'stack'} ({n} rays): " + ", ".join(
        f"{m} {n / min(v) / 1e3:.0f} Mrays/s ({min(v) * 1e3:.1f} us, x{base / min(v):.3f})" for m, v in res.items()),
        flush=True)
    h.close()
