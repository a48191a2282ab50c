"""Build every sweep format of a config and launch the trace kernel once per variant (for an
`ncu --metrics dram__bytes_read.sum,...` pass). Prints one line per launch, in launch order."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2410_14128_b200 import vf  # noqa: E402

cfg = sys.argv[1]
vol = bench.make_volume(bench.CONFIGS[cfg][0])
k, c = inputs.voxels_device(vol)
rays = torch.from_numpy(bench.make_rays(cfg)[0]).cuda()
hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
incoh = bench.CONFIGS[cfg][1] == "incoherent"
for fmt in bench.SWEEP[cfg]:
    h = vf.build((k, c, inputs.dims_of(vol)), fmt)
    for restart in (False, True):
        h.trace(rays, hits, restart=restart, incoherent=incoh)
        torch.cuda.synchronize()
        print(f"LAUNCH {cfg}|{h.signature}|{'restart' if restart else 'stack'} {rays.shape[0]}", flush=True)
    h.close()
