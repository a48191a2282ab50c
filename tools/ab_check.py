"""Bit-compare a variant library / env mode against the in-tree default kernel on full frames:
python tools/ab_check.py CFG [CFG...]   (env of the variant: VF_LIB, VF_CHUNKED, ...; runs the
default in a subprocess without them)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import bench, inputs
from paper_2410_14128_b200 import vf
cfg, out = sys.argv[1], sys.argv[2]
vol = bench.make_volume(bench.CONFIGS[cfg][0])
k, c = inputs.voxels_device(vol)
h = vf.build((k, c, inputs.dims_of(vol)), bench.CONFIGS[cfg][2])
rays = torch.from_numpy(bench.make_rays(cfg)[0]).cuda()
np.save(out, np.stack([h.trace(rays, restart=r).cpu().numpy() for r in (False, True)]))
'''
for cfg in sys.argv[1:]:
    env_v = dict(os.environ, ROOT=ROOT)
    env_d = {k: v for k, v in env_v.items() if not k.startswith("VF_")}
    outs = []
    for name, env in (("variant", env_v), ("default", env_d)):
        f = f"/tmp/abchk_{cfg}_{name}.npy"
        r = subprocess.run([sys.executable, "-c", code, cfg, f], env=env, capture_output=True, text=True)
        if r.returncode:
            print(f"{cfg} {name} FAILED: {r.stderr[-1500:]}")
            sys.exit(1)
        outs.append(np.load(f))
    same = np.array_equal(outs[0], outs[1])
    print(f"{cfg}: variant == default: {same}" + ("" if same else f" ({int((outs[0] != outs[1]).any(-1).sum())} rays differ)"))
    if not same:
        sys.exit(1)
