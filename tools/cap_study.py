import os, sys, statistics, subprocess
ROOT = "/root/repo"
code = r'''
import sys, os, statistics, torch
sys.path.insert(0, "/root/repo")
import bench, inputs
from paper_2410_14128_b200 import vf
for cfg in ("cfg4", "cfg5"):
    vname, _, fmt, _ = bench.CONFIGS[cfg]
    vol = bench.make_volume(vname)
    k, c = inputs.voxels_device(vol)
    h = vf.build((k, c, inputs.dims_of(vol)), fmt)
    del k, c
    rays = torch.from_numpy(bench.make_rays(cfg)[0]).cuda()
    hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
    flush = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
    for _ in range(3): h.trace(rays, hits)
    ms = []
    for i in range(15):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.trace(rays, hits); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    cn = h.counters(rays, hits)
    n = rays.shape[0]
    print(f"{cfg}: {statistics.median(ms):.4f} ms, {n/statistics.median(ms)/1e3:.0f} Mrays/s, capped {cn['exact_calls']/n:.4f}, tests/ray {cn['cell_tests']/n:.2f}, simt_bound {cn['cell_tests']/max(cn['warp_max_tests'],1):.3f}")
    h.close()
'''
for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, VF_LIB=lib), capture_output=True, text=True)
    print(lib, r.stdout.strip().replace("\n", " | "), r.stderr[-300:] if r.returncode else "", flush=True)
