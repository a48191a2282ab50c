"""A/B: rays regrouped into warps by their (previous-frame) iteration count inside screen tiles,
vs the plain 8x4-pixel warp tiles. The per-ray counts come from the counting run of the same
frame (tools/ray_tests_dump.py -> build/raytests/raytests_<cfg>.npy). Timing only: hits come out
in the permuted order and are compared after un-permuting.
Usage: python tools/raysort_ab.py cfg4 cfg5 cfg2"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench
import inputs
from paper_2410_14128_b200 import vf

flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")


def timeit(h, rays, hits, schedule, reps=15):
    for _ in range(3):
        h.trace(rays, hits, schedule=schedule)
    ms = []
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.trace(rays, hits, schedule=schedule)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


for cfg in sys.argv[1:]:
    vname, _, fmt, _ = bench.CONFIGS[cfg]
    vol = bench.make_volume(vname)
    k, c = inputs.voxels_device(vol)
    h = vf.build((k, c, inputs.dims_of(vol)), fmt)
    del k, c
    rays_np = bench.make_rays(cfg)[0]
    n = rays_np.shape[0]
    cost = np.load(os.path.join(ROOT, "build", "raytests", f"raytests_{cfg}.npy")).astype(np.int64)
    variants = {"natural": np.arange(n)}
    for g in (256, 1024):
        m = n // g * g
        idx = np.arange(m).reshape(-1, g)
        key = -cost[:m].reshape(-1, g)  # longest first inside the group
        o = np.take_along_axis(idx, np.argsort(key, axis=1, kind="stable"), 1).ravel()
        variants[f"sorted{g}"] = np.concatenate([o, np.arange(m, n)])
        # coarse: 4 cost classes (quartiles of the group), screen order inside a class
        q = np.floor(np.log2(cost[:m] + 1) * 2).reshape(-1, g)
        o = np.take_along_axis(idx, np.argsort(-q, axis=1, kind="stable"), 1).ravel()
        variants[f"classes{g}"] = np.concatenate([o, np.arange(m, n)])
    ref = None
    out = []
    for name, perm in variants.items():
        r = torch.from_numpy(np.ascontiguousarray(rays_np[perm])).cuda()
        hits = torch.empty((n, 4), dtype=torch.int32, device="cuda")
        t0 = timeit(h, r, hits, False)
        t1 = timeit(h, r, hits, True)
        back = torch.empty_like(hits)
        back[torch.from_numpy(perm).cuda()] = hits
        if ref is None:
            ref = back.clone()
        assert torch.equal(back, ref), name
        out.append(f"{name} {n / t0 / 1e3:.0f} / sched {n / t1 / 1e3:.0f}")
        del r
    print(f"{cfg} {fmt}: " + ", ".join(out), flush=True)
    h.close()
