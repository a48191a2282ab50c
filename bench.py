#!/usr/bin/env python3
"""bench.py — primary-ray Mrays/s through a hybrid voxel format on 1/2/4/8 B200 (BASELINE.json metric).

Default workload: cfg5 of BASELINE.json (`configs[4]`, the config the metric's "at 1/2/4/8 B200" is
quoted on) — the 4096^3 sparse procedural volume (inputs.sparse, seed 0x4096), one 3840x2160
perspective frame, format R(5^3) G(7) (the best hybrid of the cfg5 sweep, profiles/r2_pareto.md). A step = ONE
FRAME: its rays are sharded over the N GPUs by interleaved 16x16 screen tiles (tile mod N; the
volume is replicated on every GPU), every rank traces its tiles (all §8(a) rows run inside the one
trace kernel) and the hits reach rank 0's frame buffer through the one collective (north_star,
SURVEY.md §8(e)): by default fused into the trace kernel itself — vf_trace_scatter stores each hit
at its pixel in rank 0's frame over NVLink (CUDA IPC), then a one-int all-reduce signals completion
(--gather p2p); or a chunked trace + NCCL gather pipeline (--gather nccl, also the fallback). At
N = 1 the frame is one trace launch. Total work is fixed as N grows ("scaling": "strong"). Inputs are resident in HBM; L2 (126 MB) is flushed between
timed steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg5] [--format "R(5^3) G(7)"] [--restart]
                  [--sweep [--sweep-out FILE]] [--no-cpu-baseline] [--no-side]

--gpus N > 1 outside torchrun re-launches itself under torch.distributed.run (one rank per GPU);
under torchrun WORLD_SIZE must equal N. Rank 0 prints ONE compact JSON line (< 4 KB); the
per-format sweep (--sweep) goes to a file under profiles/, never into that line.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "primary-ray Mrays/s per hybrid format at 1/2/4/8 B200 vs bytes/voxel"
CONFIGS = {
    # name: (volume preset, camera preset, default format, description)
    "cfg1": ("sphere", None, "R(6, 6, 6)", "64^3 analytic sphere, Raw only, 256x256 orthographic rays"),
    "cfg2": ("menger", "menger", "G(5) R(3, 3, 3)", "256^3 Menger sponge, 1024x1024 perspective rays"),
    "cfg3": ("terrain", "terrain", "T(2, 2) T(2, 1) R(4, 4, 4)", "1024^3 noise terrain/caves, 1920x1080 rays"),
    "cfg4": ("city", "city", "R(4, 4, 4) G(7)", "2048^3 synthetic city blocks, 1920x1080 aerial rays"),
    "cfg5": ("sparse", "sparse", "R(5, 5, 5) G(7)",
             "4096^3 sparse procedural shells, 3840x2160 rays tile-sharded over the GPUs"),
    # incoherent secondary-style rays through the cfg4 city (not a BASELINE config)
    "cfg4i": ("city", "incoherent", "R(4, 4, 4) G(7)",
              "2048^3 city, 2073600 incoherent rays (uniform origins in the lower city, random directions, tmax 256)"),
    # shadow + AO rays spawned from the cfg4 primary hits (SURVEY §8(f) NEXT 3 as specified)
    "cfg4s": ("city", "secondary", "R(4, 4, 4) G(7)",
              "2048^3 city, shadow + AO rays spawned from the 1920x1080 aerial primary hits"),
    # SURVEY §8(d) cfg4 "plus a street-level view": grazing rays along the street (not a BASELINE config)
    "cfg4st": ("city", "city_street", "R(4, 4, 4) G(7)", "2048^3 city, 1920x1080 street-level view"),
    # the paper's 512^3 Table 2 rows (21-40) on a 512^3 city (not a BASELINE config)
    "t512": ("city512", "city512", "R(4, 4, 4) G(5)", "512^3 synthetic city blocks, 1024x1024 rays (Table 2 rows 21-40)"),
}
# per-config format sweeps: Mrays/s per hybrid format vs bytes/voxel
SWEEP = {
    "cfg1": ["R(6, 6, 6)", "R(3, 3, 3) R(3, 3, 3)", "G(6)", "S(6)", "T(2, 3)"],
    "cfg2": ["S(8)", "G(8)", "G(5) R(3, 3, 3)", "T(2, 4)", "R(8, 8, 8)", "R(3, 3, 3) G(5)"],
    "cfg3": ["T(2, 2) T(2, 1) R(4, 4, 4)", "T(2, 1) T(2, 2) R(4, 4, 4)", "S(5) R(5, 5, 5)", "G(10)",
             "R(3, 3, 3) G(7)", "T(2, 5)", "S(10)"],
    "cfg4": ["R(4, 4, 4) G(7)", "R(3, 3, 3) G(8)", "G(11)", "S(11)", "R(6, 6, 6) G(5)", "R(8, 8, 8) G(3)",
             "R(4, 4, 4) S(7)", "R(6, 6, 6) S(5)", "S(3) G(8)", "S(5) G(6)", "S(7) G(4)", "R(4, 4, 4) R(3, 3, 3) G(4)",
             "R(4, 4, 4) S(3) G(4)", "R(4, 4, 4) R(4, 4, 4) R(3, 3, 3)", "R(1, 1, 1) T(2, 5)", "T(2, 4) R(3, 3, 3)",
             "T(2, 2) T(2, 2) R(3, 3, 3)", "T(2, 3) R(5, 5, 5)", "R(5, 5, 5) G(6)", "D(5, 5, 5, 6) G(6)"],
    "cfg5": ["R(5, 5, 5) G(7)", "R(4, 4, 4) G(8)", "R(3, 3, 3) G(9)", "G(12)", "T(2, 6)", "S(12)", "R(4, 4, 4) T(2, 4)",
             "R(4, 4, 4) R(4, 4, 4) R(4, 4, 4)", "D(4, 4, 4, 6) G(8)", "D(3, 3, 3, 6) G(9)", "D(5, 5, 5, 6) G(7)",
             "R(6, 6, 6) G(6)", "D(6, 6, 6, 6) G(6)", "R(7, 7, 7) G(5)"],
}
# PAPER.md Table 2 (tests/golden/table2_formats.txt): rows 1-20 on cfg4, rows 21-40 on t512
_T2 = [l.strip().split(" ", 2) for l in open(os.path.join(ROOT, "tests", "golden", "table2_formats.txt"))
       if l.strip() and not l.startswith("#")]
SWEEP["cfg4"] = SWEEP["cfg4"] + [sig for _, res, sig in _T2 if res == "2048" and "D(" in sig]
SWEEP["t512"] = [sig for _, res, sig in _T2 if res == "512"]
SWEEP["cfg4i"] = ["R(4, 4, 4) G(7)", "R(3, 3, 3) G(8)", "G(11)", "S(11)", "R(6, 6, 6) G(5)", "R(1, 1, 1) T(2, 5)",
                  "D(6, 6, 6, 6) G(5)", "R(8, 8, 8) G(3)"]
SWEEP["cfg4s"] = SWEEP["cfg4i"]
L2_BYTES = 126 * 2**20
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")
HBM_FALLBACK_GBS = 7700.0  # /opt/skills/guides/B200_PROFILING.md nominal, only if MEASURED_PEAKS.json is absent


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_volume(name):
    import inputs
    return {"sphere": inputs.sphere, "menger": inputs.menger, "terrain": inputs.terrain, "city": inputs.city,
            "sparse": inputs.sparse, "city512": lambda: inputs.city(512)}[name]()


def frame_width(cfg):
    from inputs.rays import CAMERAS
    cam = CONFIGS[cfg][1]
    if cam is None:
        return 256
    if cam in ("incoherent", "secondary"):
        return 1920
    return CAMERAS[cam]["width"]


def make_rays(cfg, primary_hits=None):
    """(rays (n, 8) fp32, perm ray -> pixel). cfg4s needs the primary hits (xyz, t, normal)."""
    from inputs import rays as R
    vol, cam, _, _ = CONFIGS[cfg]
    if cam is None:
        return R.ortho(256, 256, 0.25, -1.0)
    if cam == "incoherent":
        n = 1920 * 1080
        return R.incoherent(n, (0, 16, 0), (2048, 400, 2048), 0x5EC0, tmax=256.0), np.arange(n)
    if cam == "secondary":
        prim, perm = R.camera("city")
        xyz, t, nrm = primary_hits
        rays, src = R.secondary(prim, xyz, t, nrm, seed=0x5EC1)
        return rays, perm[src]
    return R.camera(cam)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/vf_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader",
                                          "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1].split()[0]), float(f[2].split()[0]), f[4:]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, fl in rows:
            for n, v in zip(names, fl[1:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        busy = [r[0] for r in rows if r[0] > 300] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(r[1] for r in rows), "reasons": sorted(reasons),
                "samples": len(rows)}


def peaks():
    try:
        return json.load(open(MEASURED_PEAKS))
    except Exception:
        return {}


def host_cpu():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model


def oracle_grid(vol_desc):
    """The oracle's occupancy for a volume: the dense bitset when host
    memory allows (its build timed separately, §8(d) "Bitset materialisation is timed
    separately"), else the procedural occupancy (same definition, evaluated per visited cell)."""
    import oracle
    import inputs
    dims = inputs.dims_of(vol_desc)
    bits = dims[0] * dims[1] * dims[2] / 8
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    if avail > 4 * bits:
        t0 = time.perf_counter()
        g = oracle.Grid.from_generator(vol_desc)
        return g, "bitset", time.perf_counter() - t0
    return oracle.Grid.procedural(vol_desc), "procedural", 0.0


def cpu_baseline(vol_desc, rays, gpu_xyz, gpu_t, budget_s=15.0):
    """Oracle (as it stands) on the box's host cores over a bounded, evenly strided sample of the
    same frame; also checks parity of the sampled rays against the GPU hits."""
    import oracle
    from parity import compare
    g, kind, build_s = oracle_grid(vol_desc)
    cores = oracle.max_threads()
    n = len(rays)
    m = min(n, 4096)
    while True:
        idx = np.linspace(0, n - 1, m).astype(np.int64)
        t0 = time.perf_counter()
        ref = g.trace(rays[idx])
        dt = time.perf_counter() - t0
        if dt > budget_s / 4 or m >= n:
            break
        m = min(n, int(m * min(8.0, max(2.0, budget_s / max(dt, 1e-3) / 2))))
    nb, _ = compare(gpu_xyz[idx], gpu_t[idx], ref)
    g.close()
    return {"value": round(m / dt / 1e6, 4), "unit": "Mrays/s", "cores": cores, "kind": "oracle",
            "sample": f"{m} of {n} rays (evenly strided) of the frame; exact int128 DDA over the {kind} occupancy"
                      f" ({'bitset build ' + format(build_s, '.1f') + ' s, untimed' if kind == 'bitset' else 'per cell'}),"
                      f" OpenMP {cores} threads, {dt:.1f} s",
            "parity_checked": int(m), "parity_mismatches": int(nb)}


def max_over_ranks(vals, dev, dist_on):
    """Element-wise max over ranks (CUDA-event times: the frame ends when the slowest rank ends)."""
    if not dist_on:
        return list(vals)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


class FrameStep:
    """One frame on N ranks. Two forms of the one collective:
    * "p2p" (default for N > 1): the fused trace + gather — every rank's trace kernel stores its
      interleaved 16x16 tiles' hits straight into rank 0's frame buffer over NVLink / NVSwitch
      (vf_trace_scatter into a CUDA-IPC-mapped peer buffer, shard.PeerFrame), then a one-int
      all-reduce signals completion;
    * "nccl": this rank's tiles are traced in K chunks; after chunk k is traced its hit records are
      gathered to rank 0 asynchronously over NCCL, so the transfer overlaps the trace of chunk k+1
      (shard.ChunkedGather). Also the fallback when the peer mapping fails.
    With one rank (and no --force-dist) the frame is one trace launch and there is nothing to
    gather. `trace(rays_view, hits_view)` / `trace_scatter(rays, dest_ptr, slots)` launch one trace
    on the current stream."""

    def __init__(self, trace, rays_local, counts, rank, world, dist_on, device, chunks=0, timed=True,
                 trace_scatter=None, pixels_local=None, n_total=0, gather="p2p"):
        import torch
        from paper_2410_14128_b200 import shard
        self.trace, self.rays, self.timed = trace, rays_local, timed
        self.trace_scatter = trace_scatter
        self.n_local = counts[rank]
        self.pipe = self.peer = None
        self.gather = "none"
        self.gather_note = ""
        if dist_on and gather == "p2p" and trace_scatter is not None:
            try:
                self.peer = shard.PeerFrame(n_total, pixels_local, device)
                self.gather = "p2p"
            except Exception as e:  # every rank raises together (PeerFrame agrees on failure)
                self.gather_note = f"p2p unavailable ({e}); NCCL gather"
        if dist_on and self.peer is None:
            k = chunks if chunks > 0 else max(1, min(4, max(counts) // (1 << 19)))
            self.pipe = shard.ChunkedGather(counts, k, device)
            self.hits = self.pipe.hits
            self.gather = "nccl"
        elif self.peer is not None:
            self.hits = None  # the frame lives on rank 0 (pixel order); local_hits() reads it back
        else:
            self.hits = torch.empty((self.n_local, 4), dtype=torch.int32, device=device)
        self.launches = len(self.pipe.bounds) if self.pipe else 1
        self.kernel_events = []

    def _timed(self, fn, *a):
        import torch
        if self.timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*a)
            e1.record()
            self.kernel_events.append((e0, e1))
        else:
            fn(*a)

    def _trace(self, lo, hi, hv):
        self._timed(self.trace, self.rays[lo:hi], hv)

    def capture(self):
        """Single-rank frame: capture its one trace launch in a CUDA graph, replayed by every later
        call (no per-step host launch cost between the step's events; the step time is then the
        kernel's own time)."""
        import torch
        if self.pipe is not None or self.peer is not None:
            return
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.trace(self.rays[:self.n_local], self.hits)
        torch.cuda.synchronize()

    def __call__(self):
        if getattr(self, "graph", None) is not None:
            self.graph.replay()
            return None
        if self.peer is not None:
            return self.peer.run(lambda r, ptr, sl: self._timed(self.trace_scatter, r, ptr, sl), self.rays)
        if self.pipe is None:
            self._trace(0, self.n_local, self.hits)
            return None
        return self.pipe.run(self._trace)

    def launches_per_step(self, count):
        """Kernel launches of one step: count(ray view) per trace call (vf_trace_launch_count: 3 when
        VF_TRACE_SCHEDULE reorders the call, else 1)."""
        if self.pipe is None:
            return count(self.rays[:self.n_local])
        return sum(count(self.rays[lo:hi]) for lo, hi in self.pipe.bounds)

    def local_hits(self):
        """This rank's hits in its own ray order (rank 0 only in p2p mode)."""
        if self.peer is not None:
            return self.peer.frame[self.peer.slots.long()] if self.peer.frame is not None else None
        return self.hits[:self.n_local]

    def kernel_ms(self, step_ms=None):
        """Sum of the trace launches' CUDA-event durations since the last call (then reset); for a
        graph-replayed single launch, the steps' own event times (the step is that one kernel)."""
        if getattr(self, "graph", None) is not None and step_ms is not None:
            self.kernel_events = []
            return sum(step_ms)
        ms = sum(a.elapsed_time(b) for a, b in self.kernel_events)
        self.kernel_events = []
        return ms


def algorithmic_bytes(handle, rays, restart):
    """Algorithmic bytes per ray: 48 B ray I/O + the format words the traversal
    reads, counted by the counting variant of the same kernel (per-step byte table)."""
    n = rays.shape[0]
    c = handle.counters(rays, restart=restart)
    return (48 * n + c["format_bytes"]) / n, c


def build_handle(vol, fmt):
    import torch
    import inputs
    from paper_2410_14128_b200 import vf
    t0 = time.perf_counter()
    keys, rgba = inputs.voxels_device(vol)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    dims = inputs.dims_of(vol)
    vf.build((keys, rgba, dims), fmt).close()  # warm-up build (module load, first allocations)
    bts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hb = vf.build((keys, rgba, dims), fmt)
        torch.cuda.synchronize()
        bts.append(time.perf_counter() - t1)
        hb.close()
    handle = vf.build((keys, rgba, dims), fmt)
    nonempty = int(keys.shape[0])
    del keys, rgba
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return handle, nonempty, statistics.median(bts), gen_s


def side_cfg4(args, stream, flush):
    """north_star's 2048^3 target (cfg4, R(4^3) G(7), one 1920x1080 frame on this GPU): device-timed
    Mrays/s, reported beside the headline (not a bench line of its own)."""
    import torch
    vname, _, fmt, _ = CONFIGS["cfg4"]
    vol = make_volume(vname)
    h, nonempty, _, _ = build_handle(vol, fmt)
    rays_np, _ = make_rays("cfg4")
    rays = torch.from_numpy(np.ascontiguousarray(rays_np)).cuda()
    hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
    sched = {"on": True, "off": False, "regroup": "regroup"}[args.schedule]

    def timed(schedule):
        for _ in range(3):
            h.trace(rays, hits, restart=args.restart, schedule=schedule)
        ms = []
        for i in range(max(args.steps, 5)):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h.trace(rays, hits, restart=args.restart, schedule=schedule)
            b.record(stream)
            ms.append((a, b))
        torch.cuda.synchronize()
        return statistics.mean(a.elapsed_time(b) for a, b in ms)

    t = timed(sched)
    t_nat = timed(False) if sched else t
    st = h.stats()
    h.close()
    return {"workload": "cfg4: 2048^3 city, 1920x1080 aerial", "format": "R(4^3) G(7)",
            "value": round(rays.shape[0] / (t / 1e3) / 1e6, 1), "unit": "Mrays/s", "kernel_ms": round(t, 4),
            "index_order_value": round(rays.shape[0] / (t_nat / 1e3) / 1e6, 1),
            "bytes_per_voxel": round(st["bytes_used"] / nonempty, 4)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # --force-dist (test aid): run the N > 1 code path (NCCL group, chunked trace/gather pipeline,
    # max-over-ranks reductions) with a single rank
    dist_on = world > 1 or args.force_dist
    if dist_on and world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if dist_on:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2410_14128_b200 import shard

    cfg = args.config
    vname, _, deffmt, desc = CONFIGS[cfg]
    fmt = args.format or deffmt
    vol = make_volume(vname)
    handle, nonempty, build_s, gen_s = build_handle(vol, fmt)
    stats = handle.stats()
    dims = tuple(int(x) for x in vol.dims)

    prim = None
    if CONFIGS[cfg][1] == "secondary":  # secondary rays spawn from the primary hits (same API)
        from inputs import rays as R
        prays, _ = R.camera("city")
        pr = torch.from_numpy(prays).to(dev)
        ph, pp = handle.trace_payload(pr)
        torch.cuda.synchronize()
        o = ph.cpu().numpy()
        nrm = np.ascontiguousarray(pp.cpu().numpy()[:, 1]).view(np.int8).reshape(-1, 4)[:, :3]
        prim = (o[:, :3], o[:, 3].view(np.float32), nrm)
        del pr, ph, pp
    rays_all, perm = make_rays(cfg, prim)
    n_total = len(rays_all)
    width = frame_width(cfg)
    if dist_on:
        own = shard.shard(perm, width, rank, world)
        counts = shard.shard_counts(perm, width, world)
    else:
        own = np.arange(n_total)
        counts = [n_total]
    replicas = None
    if dist_on:  # §8(e) "Replicas": every rank built the same volume; compare digests over gloo
        gloo = dist.new_group(backend="gloo")
        replicas = shard.verify_replicas(shard.replica_digest(handle), group=gloo)
    rays = torch.from_numpy(np.ascontiguousarray(rays_all[own])).to(dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    incoh = CONFIGS[cfg][1] == "incoherent"  # VF_TRACE_INCOHERENT hint (not for cfg4s: its screen-ordered secondary rays are coherent enough, plain kernel +36 %)

    sched = args.schedule != "off" and not incoh  # VF_TRACE_SCHEDULE (coherent launches only)
    if sched and args.schedule == "regroup":
        sched = "regroup"  # + VF_TRACE_REGROUP (opt-in: pays only when the camera does not move)

    def trace(rv, hv):
        handle.trace(rv, hv, restart=args.restart, incoherent=incoh, schedule=sched)

    def trace_scatter(rv, ptr, slots):
        handle.trace_scatter(rv, ptr, slots, restart=args.restart, incoherent=incoh, schedule=sched)

    step = FrameStep(trace, rays, counts, rank, world, dist_on, dev, args.gather_chunks,
                     trace_scatter=trace_scatter, pixels_local=perm[own], n_total=n_total, gather=args.gather)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    step.capture()  # N = 1: the frame's one launch replayed as a CUDA graph
    step()
    torch.cuda.synchronize()
    step.kernel_ms()  # reset: only the timed steps' launches count
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev = []
    for i in range(args.steps):
        flush.fill_(i)  # write > L2 between steps (outside the step's events)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = step.kernel_ms(step_ms) / args.steps  # this rank's trace launches per step
    tot_ms, kern_max = max_over_ranks([sum(step_ms), kern_ms], dev, dist_on)
    value = n_total * args.steps / (tot_ms / 1e3) / 1e6

    # ---- end to end through the public API with HOST buffers: every rank copies its shard's rays
    # from pinned host memory, traces and copies the hits back (vf_trace_host; PCIe-bound, so its
    # chunks run in index order, no VF_TRACE_SCHEDULE); the ranks share the
    # node's host memory, so the frame's hits land on the host with no device collective. Time per
    # frame = max over ranks.
    hr = torch.from_numpy(np.ascontiguousarray(rays_all[own])).pin_memory()
    hh = torch.empty((len(own), 4), dtype=torch.int32).pin_memory()
    for _ in range(2):
        handle.trace_host(hr, hh, restart=args.restart, incoherent=incoh)
    e2e = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.fill_(1)
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        t1 = time.perf_counter()
        handle.trace_host(hr, hh, restart=args.restart, incoherent=incoh)
        e2e.append(time.perf_counter() - t1)
    e2e = max_over_ranks(e2e, dev, dist_on)
    e2e_val = n_total / statistics.median(e2e) / 1e6

    result = None
    if rank == 0:
        # roofline of the dominant (only) kernel of the step: algorithmic bytes per launch over its
        # CUDA-event duration; at N > 1 rank 0's shard and launches
        bpr, ctr = algorithmic_bytes(handle, rays, args.restart)
        kmean_ms = kern_ms / step.launches
        launch_bytes = bpr * rays.shape[0] / step.launches
        pk = peaks()
        hbm = pk.get("hbm_gbs") or HBM_FALLBACK_GBS
        key = f"{cfg}|{handle.signature}|{'restart' if args.restart else 'stack'}"
        try:
            ent = json.load(open(PROFILE_TRAFFIC)).get(key, {})
        except Exception:
            ent = {}
        achieved = launch_bytes / (kmean_ms / 1e3) / 1e9
        ent_rays = ent.get("rays") or n_total  # ncu entries without a ray count were full-frame launches
        traffic = None
        if ent.get("dram_bytes_per_launch"):
            traffic = round(ent["dram_bytes_per_launch"] / ent_rays * rays.shape[0] / step.launches)
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk.get("hbm_gbs") else "B200_PROFILING.md fallback",
                "alg_bytes_per_ray": round(bpr, 1), "kernel_ms": round(kmean_ms, 4),
                "kernel_share_of_step": round(kern_ms / (sum(step_ms) / args.steps), 3)}
        issue = None
        if ent.get("warp_inst_per_launch"):
            sm_mhz = (clk or {}).get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
            wi = ent["warp_inst_per_launch"] / ent_rays * rays.shape[0] / step.launches
            peak_i = 148 * 4 * sm_mhz * 1e6
            ach_i = wi / (kmean_ms / 1e3)
            issue = {"bound": "issue", "frac": round(ach_i / peak_i, 3), "unit": "warp-inst/s",
                     "warp_inst_per_ray": round(ent["warp_inst_per_launch"] / ent_rays, 1),
                     "threads_per_warp_inst": round(ent.get("thread_inst_per_launch", 0) / ent["warp_inst_per_launch"], 1)}
        launches_step = step.launches_per_step(
            lambda v: handle.launch_count(v, restart=args.restart, incoherent=incoh, schedule=sched))
        hits_np = step.local_hits().cpu().numpy()
        gxyz, gt = hits_np[:, :3], hits_np[:, 3].view(np.float32)
        cpu = None
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(vol, rays_all[own], gxyz, gt, budget_s=args.cpu_budget)
        result = {
            "metric": METRIC, "value": round(value, 1), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(tot_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg}: {desc}", "format": handle.signature,
                       "variant": ("restart" if args.restart else "stack") + ("+incoherent" if incoh else ""),
                       "kernel": "compiled-in" if stats.get("compiled_in") else "generic",
                       "volume": list(dims), "rays_per_frame": n_total, "nonempty_voxels": nonempty,
                       "rays_sha256": hashlib.sha256(np.ascontiguousarray(rays_all).tobytes()).hexdigest()[:16],
                       "bytes_used": stats["bytes_used"], "bytes_per_voxel": round(stats["bytes_used"] / nonempty, 4),
                       "bytes_per_voxel_paper": round(stats["paper_layout_bytes"] / nonempty, 4),
                       "hit_rate": round(float((gxyz[:, 0] >= 0).mean()), 4), "build_s": round(build_s, 3),
                       "voxel_gen_s": round(gen_s, 2), "l2": "flushed between timed steps (2x126 MB write)",
                       "schedule": ("longest-first block order from the previous frame's per-block durations "
                                    "(VF_TRACE_SCHEDULE; same camera every frame)" + (
                                        " + rays regrouped into warps by their iteration counts (VF_TRACE_REGROUP)"
                                        if sched == "regroup" else "")) if launches_step > step.launches
                       else "index order" + (" (a launch of <= 2 waves: nothing to reorder)" if sched else ""),
                       "parallelism": f"tile{world}: one frame's 16x16 tiles interleaved over {world} GPU(s), volume "
                                      f"replicated" + (
                                          ", fused trace + hit scatter into rank 0's frame over peer memory (CUDA IPC)"
                                          if step.gather == "p2p" else
                                          f", NCCL gather of hits to rank 0 in {step.launches} chunks"
                                          if dist_on else "") + (f" [{step.gather_note}]" if step.gather_note else "") + (
                                          f"; replicas verified on {replicas} rank(s) (bytes_used, buffer and "
                                          f"vf_query digests over gloo)" if replicas else "")},
            "e2e": {"value": round(e2e_val, 1), "unit": "Mrays/s", "h2d_bytes_per_step": n_total * 32,
                    "d2h_bytes_per_step": n_total * 16},
            "gpu_launches": args.steps * launches_step,
            "roofline": roof, "issue_roofline": issue, "cpu_baseline": cpu, "clocks": clk,
            "trace_only": round(n_total / (kern_max / 1e3) / 1e6, 1),
        }
        if world == 1 and sched:
            # the same frame with the blocks in index order (no schedule), for comparison; replayed
            # as a CUDA graph like the timed step, so the two differ only in the block order
            nat = []
            hv = step.hits
            handle.trace(rays, hv, restart=args.restart, incoherent=incoh)
            torch.cuda.synchronize()
            g_nat = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_nat):
                handle.trace(rays, hv, restart=args.restart, incoherent=incoh)
            for i in range(max(5, min(args.steps, 10))):
                flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g_nat.replay()
                b.record(stream)
                nat.append((a, b))
            torch.cuda.synchronize()
            nat_ms = statistics.median(a.elapsed_time(b) for a, b in nat)
            result["index_order"] = {"value": round(n_total / (nat_ms / 1e3) / 1e6, 1), "kernel_ms": round(nat_ms, 4)}
        if world == 1 and not args.no_side and cfg != "cfg4":
            result["cfg4_2048"] = side_cfg4(args, stream, flush)
        if args.sweep and world == 1 and cfg in SWEEP:
            out = args.sweep_out or os.path.join(ROOT, "profiles", f"r2_{cfg}_sweep.json")
            hb = step.hits if step.hits is not None else torch.empty((rays.shape[0], 4), dtype=torch.int32, device=dev)
            rows = sweep(cfg, vol, rays, hb, stream, flush, args)
            with open(out, "w") as f:
                json.dump({"config": cfg, "rows": rows, "clocks": clk,
                           "rays_sha256": hashlib.sha256(np.ascontiguousarray(rays_all).tobytes()).hexdigest()}, f,
                          indent=1)
            result["sweep_file"] = os.path.relpath(out, ROOT)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()
    return result


def sweep(cfg, vol, rays, hits, stream, flush, args):
    """Every format of the config's sweep: Mrays/s (stack and restart), bytes/voxel (device and
    paper layout), algorithmic bytes/ray from the counting kernel, the HBM roofline fraction, and
    parity against the oracle on a strided sample (written to a file, not the bench line)."""
    import torch
    import inputs
    import oracle
    from parity import compare
    from paper_2410_14128_b200 import vf
    keys, rgba = inputs.voxels_device(vol)
    dims = inputs.dims_of(vol)
    hbm = peaks().get("hbm_gbs") or HBM_FALLBACK_GBS
    n = rays.shape[0]
    idx = np.linspace(0, n - 1, min(n, 1 << 18)).astype(np.int64)
    g, _, _ = oracle_grid(vol)
    ref = g.trace(rays.cpu().numpy()[idx])
    g.close()
    incoh = CONFIGS[cfg][1] == "incoherent"
    out = []
    for fmt in SWEEP[cfg]:
        try:
            h = vf.build((keys, rgba, dims), fmt)
        except vf.VfError as e:
            out.append({"format": fmt, "error": str(e)})
            continue
        st = h.stats()
        no_wld = None
        if "G(" in h.signature:  # whole-level de-dup ablation: bytes only
            h2 = vf.build((keys, rgba, dims), fmt, flags=0)
            no_wld = h2.stats()["bytes_used"]
            h2.close()
        for restart in (False, True):
            c = h.counters(rays, hits[:n], restart=restart)
            alg = 48 * n + c["format_bytes"]
            for _ in range(3):
                h.trace(rays, hits[:n], restart=restart, incoherent=incoh)
            ms = []
            for i in range(7):
                flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                h.trace(rays, hits[:n], restart=restart, incoherent=incoh)
                b.record(stream)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            t_ms = statistics.median(ms)
            o = hits[:n].cpu().numpy()
            nb, _ = compare(o[idx, :3], o[idx, 3].view(np.float32), ref)
            t_sched = None
            if not incoh:  # the same frames with VF_TRACE_SCHEDULE (order from the previous frame)
                for _ in range(3):
                    h.trace(rays, hits[:n], restart=restart, schedule=True)
                ms = []
                for i in range(7):
                    flush.fill_(i)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    h.trace(rays, hits[:n], restart=restart, schedule=True)
                    b.record(stream)
                    torch.cuda.synchronize()
                    ms.append(a.elapsed_time(b))
                t_sched = statistics.median(ms)
                o = hits[:n].cpu().numpy()
                nb += compare(o[idx, :3], o[idx, 3].view(np.float32), ref)[0]
            out.append({"format": h.signature, "variant": "restart" if restart else "stack",
                        "kernel": "compiled-in" if st.get("compiled_in") else "generic",
                        "mrays_s": round(n / (t_ms / 1e3) / 1e6, 1),
                        "mrays_s_scheduled": round(n / (t_sched / 1e3) / 1e6, 1) if t_sched else None,
                        "bytes_per_voxel": round(st["bytes_used"] / st["nonempty_voxels"], 4),
                        "paper_bytes_per_voxel": round(st["paper_layout_bytes"] / st["nonempty_voxels"], 4),
                        "mib": round(st["bytes_used"] / 2**20, 1), "alg_bytes_per_ray": round(alg / n, 1),
                        "wld_reduction": round(no_wld / st["bytes_used"], 3) if no_wld else None,
                        "roofline_frac": round(alg / (t_ms / 1e3) / 1e9 / hbm, 5),
                        "cells_per_ray": round(c["cell_tests"] / n, 2), "descents_per_ray": round(c["descents"] / n, 2),
                        "simt_bound": round(c["cell_tests"] / max(c["warp_max_tests"], 1), 3),
                        "sector_bytes_per_ray": round(32 * c["sector_reads"] / n, 1),
                        "compulsory_bytes_per_ray": round(4 * c["unique_words"] / n, 2),
                        "parity_checked": int(len(idx)), "parity_mismatches": int(nb)})
        h.close()
    return out


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (this tier's reference arm),
    each step a bounded, evenly strided sample of the same frame."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    import oracle
    cfg = args.config
    vname, _, _, desc = CONFIGS[cfg]
    if CONFIGS[cfg][1] == "secondary":
        return {"impl": "reference", "unavailable": "cfg4s rays spawn from GPU primary hits; use cfg4"}
    vol = make_volume(vname)
    rays_all, _ = make_rays(cfg)
    g, kind, build_s = oracle_grid(vol)
    cores = oracle.max_threads()
    n = len(rays_all)
    m = 4096
    # size one step so K+W steps take about a minute in total
    t0 = time.perf_counter()
    g.trace(rays_all[np.linspace(0, n - 1, m).astype(np.int64)])
    per_ray = (time.perf_counter() - t0) / m
    m = int(min(n, max(1024, 60.0 / (args.steps + args.warmup) / per_ray)))
    idx = np.linspace(0, n - 1, m).astype(np.int64)
    sample = np.ascontiguousarray(rays_all[idx])
    for _ in range(args.warmup):
        g.trace(sample[: max(1, m // 8)])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        g.trace(sample)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = m * args.steps / tot / 1e6
    return {"impl": "reference", "metric": METRIC, "value": round(val, 5), "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int128-exact",
            "data": "synthetic",
            "config": {"workload": f"{cfg}: {desc}", "format": "dense occupancy (oracle, no format)",
                       "rays_per_frame": n},
            "cpu_baseline": {"value": round(val, 5), "unit": "Mrays/s", "cores": cores, "kind": "oracle",
                             "sample": f"{m} of {n} rays per step (evenly strided), {kind} occupancy"
                                       + (f" (bitset build {build_s:.1f} s, untimed)" if kind == "bitset" else "")
                                       + f"; {host_cpu()}"},
            "e2e": {"value": round(val, 5), "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args_list, n):
    """--gpus N > 1 outside torchrun: one rank per GPU under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *args_list]
    return subprocess.call(cmd)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--format", default=None)
    ap.add_argument("--restart", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="per-format sweep, written to --sweep-out")
    ap.add_argument("--sweep-out", default=None)
    ap.add_argument("--no-sweep", action="store_true", help="(default; kept for old command lines)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the cfg4 2048^3 side measurement")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--gather-chunks", type=int, default=0, help="N>1 nccl gather: trace/gather pipeline depth (0: auto)")
    ap.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                    help="N>1: fused trace + peer-memory hit scatter (p2p) or trace + NCCL gather")
    ap.add_argument("--schedule", default="on", choices=["on", "off", "regroup"],
                    help="VF_TRACE_SCHEDULE: blocks ordered by the previous frame's block durations "
                         "(regroup: + VF_TRACE_REGROUP, rays regrouped into warps by their iteration counts)")
    ap.add_argument("--force-dist", action="store_true", help="test aid: the N>1 code path with one rank")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "ours":
        if world_env is None and args.gpus > 1:
            sys.exit(relaunch(argv, args.gpus))
        if world_env is not None and int(world_env) != args.gpus and not args.force_dist:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res, separators=(",", ":")), flush=True)


if __name__ == "__main__":
    main()
