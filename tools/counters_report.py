"""Per-ray work counters (counting variant of the trace kernel) for a list of config:format specs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2410_14128_b200 import vf  # noqa: E402

cache = {}
for spec in sys.argv[1:]:
    cfg, fmt = spec.split(":", 1)
    vname, _, deffmt, _ = bench.CONFIGS[cfg]
    if cfg not in cache:
        cache.clear()
        vol = bench.make_volume(vname)
        cache[cfg] = (vol, inputs.voxels_device(vol), bench.make_rays(cfg)[0])
    vol, (k, c), rays_np = cache[cfg]
    h = vf.build((k, c, inputs.dims_of(vol)), fmt or deffmt)
    rays = torch.from_numpy(rays_np).cuda()
    for restart in (False, True):
        ct = h.counters(rays, restart=restart)
        n = ct["rays"]
        per = {kk: round(v / n, 3) for kk, v in ct.items() if kk not in ("rays",)}
        simt = ct["cell_tests"] / max(ct["warp_max_tests"], 1)
        print(f"{cfg} {h.signature:28s} {'restart' if restart else 'stack  '} simt_term={simt:.3f} "
              f"alg_B/ray={48 + ct['format_bytes'] / n:.1f} {per}", flush=True)
    h.close()
