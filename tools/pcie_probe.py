"""PCIe probe for the end-to-end path: pinned H2D / D2H bandwidth alone and concurrently (the
ceiling of vf_trace_host), and vf_trace_host time per frame for pipeline depths given in argv
(VF_HOST_CHUNKS, one fresh process each). python tools/pcie_probe.py [cfg] [chunks ...]"""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import numpy as np
    import torch
    import bench
    import inputs
    from paper_2410_14128_b200 import vf
    cfg = sys.argv[2]
    vol = bench.make_volume(bench.CONFIGS[cfg][0])
    k, c = inputs.voxels_device(vol)
    h = vf.build((k, c, inputs.dims_of(vol)), bench.CONFIGS[cfg][2])
    del k, c
    rays = bench.make_rays(cfg)[0]
    hr = torch.from_numpy(np.ascontiguousarray(rays)).pin_memory()
    hh = torch.empty((len(rays), 4), dtype=torch.int32).pin_memory()
    for _ in range(3):
        h.trace_host(hr, hh)
    ts = []
    for _ in range(15):
        torch.cuda.synchronize()
        t0 = __import__("time").perf_counter()
        h.trace_host(hr, hh)
        ts.append(__import__("time").perf_counter() - t0)
    m = statistics.median(ts)
    print(f"chunks={os.environ.get('VF_HOST_CHUNKS', 'default')}: {m * 1e3:.3f} ms/frame, "
          f"{len(rays) / m / 1e9:.3f} Grays/s e2e")
    sys.exit(0)

import torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = 1920 * 1080
a = torch.empty(n * 8, dtype=torch.float32).pin_memory()
b = torch.empty(n * 4, dtype=torch.int32).pin_memory()
da = torch.empty(n * 8, dtype=torch.float32, device="cuda")
db = torch.empty(n * 4, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        b.copy_(db, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d = timeit(lambda: da.copy_(a, non_blocking=True))
t_d2h = timeit(lambda: b.copy_(db, non_blocking=True))
t_both = timeit(both)
print(f"H2D {a.numel() * 4 / t_h2d / 1e6:.1f} GB/s, D2H {b.numel() * 4 / t_d2h / 1e6:.1f} GB/s, "
      f"concurrent {t_both:.3f} ms for {a.numel() * 4 / 1e6:.1f} MB in + {b.numel() * 4 / 1e6:.1f} MB out "
      f"-> PCIe-bound {n / t_both / 1e6:.3f} Grays/s", flush=True)
for ch in sys.argv[2:] or ["0"]:
    env = dict(os.environ)
    if ch != "0":
        env["VF_HOST_CHUNKS"] = ch
    r = subprocess.run([sys.executable, __file__, "--child", cfg], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-400:], flush=True)
