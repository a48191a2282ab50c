"""vf_trace_host frame time (cfg5 headline) with the library's cudaMalloc vs torch's caching
allocator behind the handle: python tools/e2e_alloc_probe.py [cfg]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2410_14128_b200 import vf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
vol = bench.make_volume(bench.CONFIGS[cfg][0])
k, c = inputs.voxels_device(vol)
rays = bench.make_rays(cfg)[0]
hr = torch.from_numpy(np.ascontiguousarray(rays)).pin_memory()
hh = torch.empty((len(rays), 4), dtype=torch.int32).pin_memory()
for rep in range(2):
    for alloc in ("torch", None):
        h = vf.build((k, c, inputs.dims_of(vol)), bench.CONFIGS[cfg][2], allocator=alloc)
        for _ in range(3):
            h.trace_host(hr, hh)
        ts = []
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h.trace_host(hr, hh)
            ts.append(time.perf_counter() - t0)
        print(f"[{rep}] allocator={alloc}: {len(rays) / statistics.median(ts) / 1e6:.1f} Mrays/s "
              f"(min {len(rays) / min(ts) / 1e6:.1f})", flush=True)
        h.close()
