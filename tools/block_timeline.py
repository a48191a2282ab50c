"""Launch-tail analysis (analysis build with -DVF_BLOCK_CLOCK): per-block start / end / SM of one
trace launch, and list-scheduling simulations of other block orders.
Usage: VF_LIB=build/variant_clk/libvf.so python tools/block_timeline.py --config cfg4 [--format SIG]"""
import argparse
import heapq
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
ap.add_argument("--slots", type=int, default=148 * 9)
ap.add_argument("--out", default=None)
ap.add_argument("--schedule", action="store_true", help="VF_TRACE_SCHEDULE launches")
ap.add_argument("--moved", type=float, default=0.0, help="camera moved sideways by this fraction (tools/sched_ab.py)")
ap.add_argument("--save", default=None, help="save the last run's per-block durations (us, by ray block) as .npy")
a = ap.parse_args()
vname, _, deffmt, _ = bench.CONFIGS[a.config]
vol = bench.make_volume(vname)
keys, rgba = inputs.voxels_device(vol)
h = vf.build((keys, rgba, inputs.dims_of(vol)), a.format or deffmt)
del keys, rgba
if a.moved:
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from sched_common import moved_rays, CAM
    rays = torch.from_numpy(moved_rays(CAM[a.config], a.moved)).cuda()
else:
    rays = torch.from_numpy(bench.make_rays(a.config)[0]).cuda()
hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
for _ in range(3):
    h.trace(rays, hits, restart=a.restart, schedule=a.schedule)
torch.cuda.synchronize()
path = a.out or f"/tmp/blk_{a.config}.bin"
if os.path.exists(path):
    os.remove(path)
os.environ["VF_BLOCK_CLOCK_OUT"] = path
flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
for i in range(3):
    flush.fill_(i)
    h.trace(rays, hits, restart=a.restart, schedule=a.schedule)
torch.cuda.synchronize()
del os.environ["VF_BLOCK_CLOCK_OUT"]
raw = np.fromfile(path, dtype=np.uint64)
runs = []
off = 0
while off < raw.size:
    nb = int(raw[off])
    runs.append(raw[off + 1:off + 1 + 3 * nb].reshape(nb, 3).astype(np.int64))
    off += 1 + 3 * nb


def simulate(dur, order, slots):
    """Greedy list scheduling: blocks start in `order` on the first free slot."""
    heap = [0.0] * slots
    heapq.heapify(heap)
    end = 0.0
    for i in order:
        t = heapq.heappop(heap)
        e = t + dur[i]
        end = max(end, e)
        heapq.heappush(heap, e)
    return end


print(f"{h.signature} {a.config} {'restart' if a.restart else 'stack'}{' scheduled' if a.schedule else ''}: {rays.shape[0]} rays, {runs[-1].shape[0]} blocks")
for r in runs:
    t0, t1, sm = r[:, 0], r[:, 1], r[:, 2]
    base = t0.min()
    span = (t1.max() - base) / 1e3
    dur = (t1 - t0) / 1e3
    nsm = int(sm.max()) + 1
    busy = 0.0
    for s in range(nsm):
        m = sm == s
        if not m.any():
            continue
        iv = sorted(zip((t0[m] - base) / 1e3, (t1[m] - base) / 1e3))
        cs, ce = iv[0]
        for s0, e0 in iv[1:]:
            if s0 > ce:
                busy += ce - cs
                cs, ce = s0, e0
            else:
                ce = max(ce, e0)
        busy += ce - cs
    last_start = (t0.max() - base) / 1e3
    dec = np.array_split(dur, 10)
    print(f"  span {span:.1f} us, SM active {busy / nsm / span:.3f}, last block starts at {last_start:.1f} us "
          f"({last_start / span:.3f}); block us mean {dur.mean():.1f} p50 {np.median(dur):.1f} p99 "
          f"{np.percentile(dur, 99):.1f} max {dur.max():.1f}")
print("  block-duration deciles by block index (us): " + " ".join(f"{d.mean():.1f}" for d in dec))
n = dur.size
if a.save and not a.schedule:
    np.save(a.save, dur)
orig = simulate(dur, range(n), a.slots)
lpt = simulate(dur, np.argsort(-dur, kind="stable"), a.slots)
rev = simulate(dur, range(n - 1, -1, -1), a.slots)
# a static interleave (block b -> tile (b * stride) mod n)
stride = 1009 if n % 1009 else 1013
inter = simulate(dur, [(b * stride) % n for b in range(n)], a.slots)
lb = max(dur.sum() / a.slots, dur.max())
print(f"  simulated makespan (us): measured-order {orig:.1f}, LPT {lpt:.1f}, reversed {rev:.1f}, "
      f"interleaved {inter:.1f}, lower bound {lb:.1f}")
