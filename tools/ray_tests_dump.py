"""Per-ray cell tests of the counting run (analysis build: tools/build_variant.sh raytests -DVF_RAY_TESTS;
then VF_LIB=build/variant_raytests/libvf.so python tools/ray_tests_dump.py) -> gpurun_out/raytests_<cfg>.npy,
the input of the block-compaction simulation in DESIGN.md §11."""
import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench, inputs
from paper_2410_14128_b200 import vf
for cfg in (sys.argv[1:] or ("cfg4", "cfg5", "cfg3", "cfg2")):
    vname, _, fmt, _ = bench.CONFIGS[cfg]
    vol = bench.make_volume(vname)
    k, c = inputs.voxels_device(vol)
    h = vf.build((k, c, inputs.dims_of(vol)), fmt)
    del k, c
    rays = torch.from_numpy(bench.make_rays(cfg)[0]).cuda()
    hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
    h.counters(rays, hits)
    np.save(f"/root/repo/gpurun_out/raytests_{cfg}.npy", hits[:, 0].cpu().numpy())
    h.close()
    print(cfg, "ok", flush=True)
