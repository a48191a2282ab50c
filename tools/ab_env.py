"""A/B of trace launch modes selected by environment variables, each in a fresh process:
python tools/ab_env.py CFG:FORMAT 'NAME=ENV1=v,ENV2=v;persistent' ...
Prints median Mrays/s (stack and restart) per mode, alternating modes twice."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, statistics, torch
import numpy as np
sys.path.insert(0, os.environ["ROOT"])
import bench, inputs
from paper_2410_14128_b200 import vf
cfg, fmt = sys.argv[1].split(":", 1)
pers = sys.argv[2] == "1"
inc = sys.argv[2] == "2"
vname, _, deffmt, _ = bench.CONFIGS[cfg]
vol = bench.make_volume(vname)
k, c = inputs.voxels_device(vol)
fl = vf.VF_BUILD_DEFAULT | (vf.VF_BUILD_ALIGN_NODES if os.environ.get("VF_AB_ALIGN") else 0)
h = vf.build((k, c, inputs.dims_of(vol)), fmt or deffmt, flags=fl)
mib = h.stats()["bytes_used"] / 2**20
del k, c
prim = None
if bench.CONFIGS[cfg][1] == "secondary":  # cfg4s: spawn from the primary hits (as bench.py does)
    from inputs import rays as R
    pr = torch.from_numpy(R.camera("city")[0]).cuda()
    ph, pp = h.trace_payload(pr)
    torch.cuda.synchronize()
    o = ph.cpu().numpy()
    nrm = np.ascontiguousarray(pp.cpu().numpy()[:, 1]).view(np.int8).reshape(-1, 4)[:, :3]
    prim = (o[:, :3], o[:, 3].view(np.float32), nrm)
rays = torch.from_numpy(bench.make_rays(cfg, prim)[0]).cuda()
hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
res = []
for restart in (False, True):
    for _ in range(3): h.trace(rays, hits, restart=restart, persistent=pers, incoherent=inc)
    ms = []
    for i in range(15):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.trace(rays, hits, restart=restart, persistent=pers, incoherent=inc); b.record()
        torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    res.append(rays.shape[0] / statistics.median(ms) / 1e3)
print(f"stack {res[0]:.0f} restart {res[1]:.0f} ({mib:.1f} MiB)")
'''
spec = sys.argv[1]
modes = sys.argv[2:]
for rep in range(2):
    for m in modes:
        name, _, rest = m.partition("=")
        envs, _, flag = rest.partition(";")
        env = dict(os.environ, ROOT=ROOT)
        for kv in filter(None, envs.split(",")):
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", code, spec, {"persistent": "1", "incoherent": "2"}.get(flag, "0")], env=env,
                           capture_output=True, text=True)
        print(f"[{rep}] {spec} {name}: {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
