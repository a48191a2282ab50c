#!/usr/bin/env python3
"""bench.py — primary-ray Mrays/s through a hybrid voxel format on B200 (BASELINE.json metric).

Default workload (N=1): cfg4 of BASELINE.json — the 2048^3 voxelised-synthetic city (TEX=1,
inputs.city), 1920x1080 aerial perspective rays, format R(4^3) G(7) (the paper's always-Pareto
2048^3 format). A step = one vf_trace of the whole frame (all §8(a) rows run inside
the one trace kernel); inputs are resident in HBM; L2 (126 MB) is flushed between timed steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg4] [--format "R(4^3) G(7)"] [--restart] [--no-sweep]

Multi-GPU (torchrun, one rank per GPU): the volume is replicated and every rank traces a whole
frame per step — rays are independent, so there is no collective in the step (weak scaling,
value = all ranks' rays / max-over-ranks time). The north_star's single frame split over the GPUs
by interleaved 16x16 screen tiles with the NCCL hit gather to rank 0 is reported beside it as
`strong_frame` (frame rate, trace-only rate).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (volume preset, camera preset, default format, description)
    "cfg1": ("sphere", None, "R(6, 6, 6)", "64^3 analytic sphere, Raw only, 256x256 orthographic rays"),
    "cfg2": ("menger", "menger", "G(5) R(3, 3, 3)", "256^3 Menger sponge, 1024x1024 perspective rays"),
    "cfg3": ("terrain", "terrain", "T(2, 2) T(2, 1) R(4, 4, 4)", "1024^3 noise terrain/caves, 1920x1080 rays"),
    "cfg4": ("city", "city", "R(4, 4, 4) G(7)", "2048^3 synthetic city blocks, 1920x1080 aerial rays"),
    "cfg5": ("sparse", "sparse", "R(4, 4, 4) G(8)", "4096^3 sparse shells, 3840x2160 rays"),
    # incoherent secondary-style rays through the cfg4 city (not a BASELINE config)
    "cfg4i": ("city", "incoherent", "R(4, 4, 4) G(7)", "2048^3 city, 2073600 incoherent rays (uniform origins in the lower city, random directions, tmax 256)"),
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
             "T(2, 2) T(2, 2) R(3, 3, 3)", "T(2, 3) R(5, 5, 5)"],
    "cfg5": ["R(4, 4, 4) G(8)", "R(3, 3, 3) G(9)", "G(12)", "T(2, 6)", "S(12)", "R(4, 4, 4) T(2, 4)",
             "R(4, 4, 4) R(4, 4, 4) R(4, 4, 4)"],
}
# PAPER.md Table 2 (tests/golden/table2_formats.txt): rows 1-20 on cfg4, rows 21-40 on t512
_T2 = [l.strip().split(" ", 2) for l in open(os.path.join(ROOT, "tests", "golden", "table2_formats.txt"))
       if l.strip() and not l.startswith("#")]
SWEEP["cfg4"] = SWEEP["cfg4"] + [sig for _, res, sig in _T2 if res == "2048" and
                                 "D(" in sig]  # the DF rows (the others are already in the list)
SWEEP["t512"] = [sig for _, res, sig in _T2 if res == "512"]
SWEEP["cfg4i"] = ["R(4, 4, 4) G(7)", "R(3, 3, 3) G(8)", "G(11)", "S(11)", "R(6, 6, 6) G(5)", "R(1, 1, 1) T(2, 5)",
                  "D(6, 6, 6, 6) G(5)", "R(8, 8, 8) G(3)"]
L2_BYTES = 126 * 2**20
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_volume(name):
    import inputs
    return {"sphere": inputs.sphere, "menger": inputs.menger, "terrain": inputs.terrain, "city": inputs.city,
            "sparse": inputs.sparse, "city512": lambda: inputs.city(512)}[name]()


def make_rays(cfg):
    from inputs import rays as R
    vol, cam, _, _ = CONFIGS[cfg]
    if cam is None:
        return R.ortho(256, 256, 0.25, -1.0)
    if cam == "incoherent":
        n = 1920 * 1080
        return R.incoherent(n, (0, 16, 0), (2048, 400, 2048), 0x5EC0, tmax=256.0), np.arange(n)
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


def cpu_baseline(vol_desc, rays, gpu_xyz, gpu_t, budget_s=12.0):
    """Oracle (as it stands) on the box's host cores over a bounded, evenly strided sample of the
    same frame; also checks parity of the sampled rays against the GPU hits."""
    import oracle
    from parity import compare
    g = oracle.Grid.procedural(vol_desc)
    cores = oracle.max_threads()
    n = len(rays)
    m = min(n, 2048)
    total_s, done, checked, bad = 0.0, 0, 0, 0
    while True:
        idx = np.linspace(0, n - 1, m).astype(np.int64)
        t0 = time.perf_counter()
        ref = g.trace(rays[idx])
        dt = time.perf_counter() - t0
        nb, _ = compare(gpu_xyz[idx], gpu_t[idx], ref)
        checked, bad = m, nb
        total_s, done = dt, m
        if dt > budget_s / 4 or m >= n:
            break
        m = min(n, int(m * min(8.0, max(2.0, budget_s / max(dt, 1e-3) / 2))))
    return {"value": done / total_s / 1e6, "unit": "Mrays/s", "cores": cores, "kind": "oracle",
            "sample": f"{done} of {n} rays (evenly strided) of the same frame; exact int128 DDA over the "
                      f"procedural occupancy (vg_voxel per visited cell), OpenMP {cores} threads; {total_s:.2f} s",
            "parity_checked": checked, "parity_mismatches": bad}, idx, ref


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
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if dist_on:
        # bind the NCCL communicator to this rank's GPU up front (barriers / collectives use it)
        dist.init_process_group("nccl", device_id=dev)
    import inputs
    from paper_2410_14128_b200 import vf

    cfg = args.config
    vname, _, deffmt, desc = CONFIGS[cfg]
    fmt = args.format or deffmt
    vol = make_volume(vname)
    t0 = time.perf_counter()
    keys, rgba = inputs.voxels_device(vol)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    dims = inputs.dims_of(vol)
    # vf_build timed alone (build throughput as a number of its own): one
    # warm-up build (first-call allocations, module load), then the median of 3 builds
    vf.build((keys, rgba, dims), fmt).close()
    bts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hb = vf.build((keys, rgba, dims), fmt)
        torch.cuda.synchronize()
        bts.append(time.perf_counter() - t1)
        hb.close()
    handle = vf.build((keys, rgba, dims), fmt)
    torch.cuda.synchronize()
    build_s = statistics.median(bts)
    nonempty = keys.shape[0]
    del keys, rgba
    torch.cuda.empty_cache()
    stats = handle.stats()

    rays_all, perm = make_rays(cfg)
    from inputs.rays import CAMERAS
    from paper_2410_14128_b200 import shard
    cam = CONFIGS[cfg][1]
    width = 256 if cam is None else (1920 if cam == "incoherent" else CAMERAS[cam]["width"])
    # The timed step (every N): each rank traces a whole frame — the rays of a frame are
    # independent, so N GPUs trace N frames with no collective in the step (weak scaling; value =
    # all ranks' rays / the max-over-ranks time). The north_star's split of ONE frame over the N
    # GPUs by 16x16 screen tiles with the NCCL hit gather is measured after it (`strong_frame`).
    own = np.arange(len(rays_all))
    rays = torch.from_numpy(np.ascontiguousarray(rays_all)).to(dev)
    n_local = rays.shape[0]
    hits = torch.empty((n_local, 4), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)

    incoh = CONFIGS[cfg][1] == "incoherent"  # VF_TRACE_INCOHERENT hint for secondary-style rays

    def step():
        handle.trace(rays, hits, restart=args.restart, incoherent=incoh)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i)  # write > L2 between steps (outside the step's events)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]  # one trace launch per step
    tot_ms = sum(kern_ms)
    if dist_on:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    n_total = len(rays_all)
    value = world * n_total * args.steps / (tot_ms / 1e3) / 1e6

    strong = None
    if dist_on:
        # One frame split over the N GPUs (interleaved 16x16 tiles, tile mod N) and its hits
        # gathered to rank 0 with NCCL, pipelined over K row chunks: K =
        # --gather-chunks, or auto, one chunk per 512k local rays (at most 4) — a trace launch
        # lasts at least as long as its slowest ray, so smaller chunks lose more in launch tails
        # than the overlap with the gather returns. Frame time = max over ranks (CUDA events).
        sh = shard.shard(perm, width, rank, world)
        rays_sh = torch.from_numpy(np.ascontiguousarray(rays_all[sh])).to(dev)
        counts = shard.shard_counts(perm, width, world)
        k_chunks = args.gather_chunks if args.gather_chunks > 0 else max(1, min(4, max(counts) // (1 << 19)))
        pipe = shard.ChunkedGather(counts, k_chunks, dev)

        def frame():
            pipe.run(lambda lo, hi, hv: handle.trace(rays_sh[lo:hi], hv, restart=args.restart, incoherent=incoh))

        for _ in range(args.warmup):
            frame()
        torch.cuda.synchronize()
        dist.barrier()
        fr, tr = [], []
        for i in range(args.steps):
            flush.fill_(i)
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(stream)
            frame()
            b.record(stream)
            handle.trace(rays_sh, pipe.hits[:rays_sh.shape[0]], restart=args.restart, incoherent=incoh)
            c.record(stream)
            fr.append((a, b))
            tr.append((b, c))
        torch.cuda.synchronize()
        t = torch.tensor([sum(x.elapsed_time(y) for x, y in fr), sum(x.elapsed_time(y) for x, y in tr)],
                         dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        strong = {"value": round(n_total * args.steps / (float(t[0]) / 1e3) / 1e6, 2), "unit": "Mrays/s",
                  "trace_only": round(n_total * args.steps / (float(t[1]) / 1e3) / 1e6, 2),
                  "gather_chunks": len(pipe.bounds), "gpu_launches_per_frame": len(pipe.bounds),
                  "note": "one frame split over the N GPUs by interleaved 16x16 tiles, hits gathered to rank 0 "
                          "with NCCL (north_star); trace_only = the same shards without the gather; max over ranks"}

    # ---- end to end through the public API with host buffers (pinned), every rank on its frame:
    # host->device copy of the rays, trace, device->host copy of the hits (vf_trace_host); the
    # time per frame is the max over ranks
    hr = torch.from_numpy(np.ascontiguousarray(rays_all)).pin_memory()
    hh = torch.empty((n_local, 4), dtype=torch.int32).pin_memory()
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
        dt = time.perf_counter() - t1
        if dist_on:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e.append(dt)
    e2e_val = world * n_total / statistics.median(e2e) / 1e6

    result = None
    if rank == 0:
        # ---- roofline: algorithmic bytes per launch / measured kernel time (trace kernel)
        kmean = statistics.mean(kern_ms)
        alg = algorithmic_bytes(handle, rays, args.restart, n_local)
        pk = peaks()
        hbm = pk.get("hbm_gbs")
        traffic = None
        try:
            tj = json.load(open(PROFILE_TRAFFIC))
            key = f"{cfg}|{handle.signature}|{'restart' if args.restart else 'stack'}"
            if key in tj:
                traffic = tj[key]["dram_bytes_per_launch"]
        except Exception:
            pass
        achieved = alg["bytes_per_launch"] / (kmean / 1e3) / 1e9
        # issue roofline: warp instructions per launch (ncu smsp__inst_executed.sum, same kernel
        # and workload) / measured kernel time vs 148 SMs x 4 schedulers x 1 warp-inst / cycle
        issue = None
        try:
            tj = json.load(open(PROFILE_TRAFFIC))
            ent = tj.get(f"{cfg}|{handle.signature}|{'restart' if args.restart else 'stack'}", {})
            wi = ent.get("warp_inst_per_launch")
            if wi:
                sm_mhz = (clk or {}).get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
                peak_i = 148 * 4 * sm_mhz * 1e6
                ach_i = wi / (kmean / 1e3)
                issue = {"bound": "issue", "achieved": round(ach_i / 1e9, 2), "peak": round(peak_i / 1e9, 2),
                         "unit": "Gwarp-inst/s", "frac": round(ach_i / peak_i, 4),
                         "warp_inst_per_ray": round(wi / n_local, 1),
                         "simt_threads_per_inst": round(ent.get("thread_inst_per_launch", 0) / wi, 2)}
        except Exception:
            pass
        roof = {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 5) if hbm else None, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if hbm else "missing",
                "algorithmic_bytes_per_ray": round(alg["bytes_per_ray"], 2), "kernel_ms": round(kmean, 4),
                "sector_bytes_per_ray": round(32 * alg.get("sector_reads", 0) / n_local, 1),
                "compulsory_bytes_per_ray": round(4 * alg.get("unique_words", 0) / n_local, 2),
                "compulsory_sector_bytes_per_ray": round(32 * alg.get("unique_sectors", 0) / n_local, 2),
                "note": "pointer-chasing; latency/issue-bound, see profiles/"}

        # ---- CPU baseline (oracle) on a bounded sample + parity of the sample
        hits_np = hits[:n_local].cpu().numpy()
        gxyz, gt = hits_np[:, :3], hits_np[:, 3].view(np.float32)
        cpu, ref_idx, ref = None, None, None
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        if not args.no_cpu_baseline and world == 1:
            cpu, ref_idx, ref = cpu_baseline(vol, rays_all, gxyz, gt, budget_s=args.cpu_budget)

        hit_rate = float((gxyz[:, 0] >= 0).mean())
        bpv = stats["bytes_used"] / max(nonempty, 1)
        result = {
            "metric": "primary-ray Mrays/s per hybrid format vs bytes/voxel",
            "value": round(value, 2), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg}: {desc}", "format": handle.signature, "variant":
                       ("restart" if args.restart else "stack") + ("+incoherent" if incoh else ""), "volume": list(dims), "rays": n_total,
                       "nonempty_voxels": int(nonempty), "bytes_used": stats["bytes_used"],
                       "paper_layout_bytes": stats["paper_layout_bytes"], "bytes_per_voxel": round(bpv, 4),
                       "bytes_per_voxel_paper": round(stats["paper_layout_bytes"] / max(nonempty, 1), 4),
                       "hit_rate": round(hit_rate, 4), "build_s": round(build_s, 4), "voxel_gen_s": round(gen_s, 3),
                       "build_mvoxels_per_s": round(nonempty / build_s / 1e6, 1),
                       "l2": "flushed between timed steps (write 2x126 MB)",
                       "parallelism": f"dp{world}: one frame per GPU, volume replicated, no collective in the step; "
                                      f"strong_frame: one frame's 16x16 tiles interleaved over {world} GPU(s) + NCCL hit gather"},
            "e2e": {"value": round(e2e_val, 2), "unit": "Mrays/s", "h2d_bytes_per_step": world * n_total * 32,
                    "d2h_bytes_per_step": world * n_total * 16},
            "strong_frame": strong,
            "gpu_launches": args.steps,
            "roofline": roof,
            "issue_roofline": issue,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        if not args.no_sweep and world == 1 and cfg in SWEEP:
            result["sweep"] = sweep(cfg, vol, rays, hits, stream, flush, args, ref_idx, ref)
    if dist_on:
        dist.destroy_process_group()
    return result


def algorithmic_bytes(handle, rays, restart, n):
    """Algorithmic bytes per launch: 48 B ray I/O per ray + format words read per ray as counted by
    the counters build of the same kernel (SURVEY.md §8(d) per-step byte table)."""
    c = handle.counters(rays, restart=restart) if hasattr(handle, "counters") else None
    if c is None:
        return {"bytes_per_launch": 48 * n, "bytes_per_ray": 48.0}
    b = 48 * n + c["format_bytes"]
    return {"bytes_per_launch": b, "bytes_per_ray": b / n, **c}


def sweep(cfg, vol, rays, hits, stream, flush, args, ref_idx=None, ref=None):
    """Every format of the config's sweep: Mrays/s (stack and restart), bytes/voxel (device and
    paper layout), algorithmic bytes/ray from the counting kernel, the HBM roofline fraction, and
    parity of the oracle-checked sample (the same rays the cpu_baseline leg traced)."""
    import torch
    import inputs
    from parity import compare
    from paper_2410_14128_b200 import vf
    keys, rgba = inputs.voxels_device(vol)
    dims = inputs.dims_of(vol)
    hbm = peaks().get("hbm_gbs")
    try:
        traffic = json.load(open(PROFILE_TRAFFIC))
    except Exception:
        traffic = {}
    out = []
    n = rays.shape[0]
    incoh = CONFIGS[cfg][1] == "incoherent"
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
            c = h.counters(rays, hits, restart=restart)
            alg = 48 * n + c["format_bytes"]
            for _ in range(3):
                h.trace(rays, hits, restart=restart, incoherent=incoh)
            ms = []
            for i in range(7):
                flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                h.trace(rays, hits, restart=restart, incoherent=incoh)
                b.record(stream)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            t_ms = statistics.median(ms)
            variant = "restart" if restart else "stack"
            row = {"format": h.signature, "variant": variant, "mrays_s": round(n / (t_ms / 1e3) / 1e6, 1),
                   "bytes_per_voxel": round(st["bytes_used"] / st["nonempty_voxels"], 4),
                   "paper_bytes_per_voxel": round(st["paper_layout_bytes"] / st["nonempty_voxels"], 4),
                   "mib": round(st["bytes_used"] / 2**20, 1), "alg_bytes_per_ray": round(alg / n, 1),
                   "wld_reduction": round(no_wld / st["bytes_used"], 3) if no_wld else None,
                   "roofline_frac": round(alg / (t_ms / 1e3) / 1e9 / hbm, 5) if hbm else None,
                   "cells_per_ray": round(c["cell_tests"] / n, 2), "descents_per_ray": round(c["descents"] / n, 2),
                   "simt_bound": round(c["cell_tests"] / max(c["warp_max_tests"], 1), 3),
                   # sector bytes (32 B x sectors spanned per load) and the frame's
                   # compulsory format bytes (distinct words read, touch bitmap) per ray
                   "sector_bytes_per_ray": round(32 * c["sector_reads"] / n, 1),
                   "compulsory_bytes_per_ray": round(4 * c["unique_words"] / n, 2),
                   "compulsory_sector_bytes_per_ray": round(32 * c["unique_sectors"] / n, 2)}
            key = f"{cfg}|{h.signature}|{variant}"
            if key in traffic:
                row["dram_bytes_per_ray"] = round(traffic[key]["dram_bytes_per_launch"] / n, 1)
            if ref is not None:
                o = hits.cpu().numpy()
                nb, _ = compare(o[ref_idx, :3], o[ref_idx, 3].view(np.float32), ref)
                row["parity_mismatches"] = nb
                row["parity_checked"] = int(len(ref_idx))
            out.append(row)
        h.close()
    return out


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (this tier's reference arm)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    import oracle
    cfg = args.config
    vname, _, deffmt, desc = CONFIGS[cfg]
    vol = make_volume(vname)
    rays_all, _ = make_rays(cfg)
    g = oracle.Grid.procedural(vol)
    cores = oracle.max_threads()
    n = len(rays_all)
    m = 4096
    # size one step so K+W steps take about a minute in total
    t0 = time.perf_counter()
    g.trace(rays_all[np.linspace(0, n - 1, m).astype(np.int64)])
    dt = time.perf_counter() - t0
    per_ray = dt / m
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
    return {"impl": "reference", "metric": "primary-ray Mrays/s per hybrid format vs bytes/voxel",
            "value": round(val, 5), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int128-exact", "data": "synthetic",
            "config": {"workload": f"{cfg}: {desc}", "format": "dense occupancy (oracle, no format)", "rays": n},
            "cpu_baseline": {"value": round(val, 5), "unit": "Mrays/s", "cores": cores, "kind": "oracle",
                             "sample": f"{m} of {n} rays per step (evenly strided), procedural occupancy"},
            "e2e": {"value": round(val, 5), "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--format", default=None)
    ap.add_argument("--restart", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the per-format sweep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--gather-chunks", type=int, default=0, help="N>1: trace/gather pipeline depth (0: auto)")
    ap.add_argument("--force-dist", action="store_true", help="test aid: the N>1 code path with one rank")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
