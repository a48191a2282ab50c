"""Quick probe of extra formats on a config: counters (cell tests, descents, pops per ray), bytes,
compiled-in or generic, Mrays/s index order and scheduled. python tools/fmt_probe.py cfg5 'FMT' ..."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
import inputs
from paper_2410_14128_b200 import vf

cfg = sys.argv[1]
vname = bench.CONFIGS[cfg][0]
vol = bench.make_volume(vname)
k, c = inputs.voxels_device(vol)
rays = torch.from_numpy(bench.make_rays(cfg)[0]).cuda()
n = rays.shape[0]
hits = torch.empty((n, 4), dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
for fmt in sys.argv[2:]:
    try:
        h = vf.build((k, c, inputs.dims_of(vol)), fmt)
    except vf.VfError as e:
        print(fmt, "error", e)
        continue
    st = h.stats()
    ct = h.counters(rays, hits)
    res = []
    for sched in (False, True):
        for _ in range(3):
            h.trace(rays, hits, schedule=sched)
        ms = []
        for i in range(9):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            h.trace(rays, hits, schedule=sched)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        res.append(n / statistics.median(ms) / 1e3)
    print(f"{h.signature:32s} {'compiled' if st['compiled_in'] else 'generic ':8s} B/vox {st['bytes_used'] / st['nonempty_voxels']:.4f} "
          f"cells {ct['cell_tests'] / n:5.1f} desc {ct['descents'] / n:4.1f} pops {ct['pops'] / n:4.1f} "
          f"steps {ct['steps'] / n:5.1f}  {res[0]:6.0f} / sched {res[1]:6.0f} Mrays/s", flush=True)
    h.close()
