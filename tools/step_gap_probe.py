"""Where do the ~10 us between a bench step's events and its trace kernel come from? Times one cfg
frame per step (L2 flushed between steps, like bench.py) in several host-side forms.
python tools/step_gap_probe.py [cfg]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2410_14128_b200 import vf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
vol = bench.make_volume(bench.CONFIGS[cfg][0])
k, c = inputs.voxels_device(vol)
h = vf.build((k, c, inputs.dims_of(vol)), bench.CONFIGS[cfg][2])
del k, c
rays = torch.from_numpy(bench.make_rays(cfg)[0]).cuda()
hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
flush = torch.empty(2 * bench.L2_BYTES // 4, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
n = rays.shape[0]


def run(name, body, steps=20, sampler=False):
    for _ in range(3):
        body()
    torch.cuda.synchronize()
    cs = bench.ClockSampler(0) if sampler else None
    if cs:
        cs.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i)
        ev[i][0].record(s)
        body()
        ev[i][1].record(s)
    torch.cuda.synchronize()
    if cs:
        cs.stop()
    ms = [a.elapsed_time(b) for a, b in ev]
    print(f"{cfg} {name:32s} median {statistics.median(ms) * 1e3:8.1f} us  mean {statistics.mean(ms) * 1e3:8.1f} us "
          f"-> {n / statistics.mean(ms) / 1e3:.0f} Mrays/s", flush=True)


run("direct trace", lambda: h.trace(rays, hits))
run("direct trace + clock sampler", lambda: h.trace(rays, hits), sampler=True)
st = bench.FrameStep(lambda rv, hv: h.trace(rv, hv), rays, [n], 0, 1, False, torch.device("cuda", 0))
run("FrameStep (bench)", st)
run("FrameStep + clock sampler", st, sampler=True)
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(s)
with torch.cuda.stream(side):
    h.trace(rays, hits, stream=side)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        h.trace(rays, hits, stream=side)
torch.cuda.synchronize()
run("CUDA graph replay", lambda: g.replay())
