"""Full-frame GPU parity at BASELINE.json's full sizes: EVERY ray of each
config's frame, in the launch configuration bench.py times, against the oracle walking the dense
occupancy bitset with OpenMP on the box's host cores.

Bar (north_star; tests/parity.py): hit voxel and miss flag bit-exact, t within 1e-4 relative.
"""
from __future__ import annotations

import functools

import numpy as np
import pytest

import inputs
import oracle
from parity import assert_parity

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=2)
def _frame(cfg):
    """(volume, rays, perm, oracle result over the whole frame) — one bitset per volume."""
    import bench
    vol = bench.make_volume(bench.CONFIGS[cfg][0])
    rays, perm = bench.make_rays(cfg)
    g = oracle.Grid.from_generator(vol)
    ref = g.trace(rays)
    g.close()
    assert (ref["status"] != 2).all()
    return vol, rays, perm, ref


def _handles(vol, fmts):
    import torch
    from paper_2410_14128_b200 import vf
    keys, rgba = inputs.voxels_device(vol)
    for fmt in fmts:
        h = vf.build((keys, rgba, inputs.dims_of(vol)), fmt)
        yield fmt, h
        h.close()
    del keys, rgba
    torch.cuda.empty_cache()


def _check(cfg, fmts, incoherent=False):
    import torch
    vol, rays, _, ref = _frame(cfg)
    rt = torch.from_numpy(rays).cuda()
    hits = torch.empty((len(rays), 4), dtype=torch.int32, device="cuda")
    for fmt, h in _handles(vol, fmts):
        for restart in (False, True):
            # as bench.py launches it: VF_TRACE_SCHEDULE for coherent rays — the first launch over the
            # array runs in index order and records block durations, the second runs reordered
            for launch in range(1 if incoherent else 2):
                h.trace(rt, hits, restart=restart, incoherent=incoherent, schedule=not incoherent)
                out = hits.cpu().numpy()
                assert_parity(out[:, :3], out[:, 3].view(np.float32), ref,
                              f"{cfg} {fmt} restart={restart} launch {launch} (full frame)")


def test_cfg1_full_frame():
    import bench
    _check("cfg1", bench.SWEEP["cfg1"])


def test_cfg2_full_frame():
    import bench
    _check("cfg2", bench.SWEEP["cfg2"])


def test_cfg3_full_frame():
    import bench
    _check("cfg3", bench.SWEEP["cfg3"])


def test_cfg4_full_frame():
    import bench
    _check("cfg4", list(dict.fromkeys(bench.SWEEP["cfg4"] + ["R(11, 11, 11)"])))


def test_cfg4i_full_frame():
    import bench
    _check("cfg4i", bench.SWEEP["cfg4i"], incoherent=True)


def test_cfg4s_secondary_full_frame():
    """SURVEY §8(f) NEXT 3 as specified: shadow + AO rays spawned from the cfg4 primary hits
    (inputs.rays.secondary; origin on the entry face from the hit voxel / t / entry-face normal).
    The spawn inputs are the ORACLE's primary hits (never the CUDA path's); every secondary ray of
    the frame is traced on the GPU in bench.py's launch configuration (plain kernel) and with the
    VF_TRACE_INCOHERENT kernel, and compared with the oracle, for every format of the cfg4s sweep,
    stack and restart."""
    import bench
    import torch
    from inputs import rays as R
    vol, prim, _, pref = _frame("cfg4")
    rays, _src = R.secondary(prim, pref["xyz"], pref["t"], pref["normal"], seed=0x5EC1)
    assert len(rays) > 1_000_000  # ~2 x the 56 % primary hit rate of 2,073,600 rays
    g = oracle.Grid.from_generator(vol)
    ref = g.trace(rays)
    g.close()
    assert (ref["status"] != 2).all()
    shadow = ref["xyz"][: len(rays) // 2, 0] >= 0
    assert 0.01 < shadow.mean() < 0.99  # both lit and shadowed points in the frame
    rt = torch.from_numpy(rays).cuda()
    hits = torch.empty((len(rays), 4), dtype=torch.int32, device="cuda")
    for fmt, h in _handles(vol, bench.SWEEP["cfg4s"]):
        for restart in (False, True):
            for incoh in (False, True):  # bench.py's launch (plain, scheduled) and the VF_TRACE_INCOHERENT kernel
                for launch in range(1 if incoh else 2):
                    h.trace(rt, hits, restart=restart, incoherent=incoh, schedule=not incoh)
                    out = hits.cpu().numpy()
                    assert_parity(out[:, :3], out[:, 3].view(np.float32), ref,
                                  f"cfg4s {fmt} restart={restart} incoherent={incoh} launch {launch} (full frame)")


def test_cfg5_full_frame_every_sweep_format():
    """cfg5 (4096^3, 3840x2160 = 8,294,400 rays): the bench's headline R(5^3) G(7) and every other
    format of the cfg5 sweep, each over the whole frame, stack and restart."""
    import bench
    _check("cfg5", bench.SWEEP["cfg5"])


def test_cfg5_tile_sharded_frame_assembled(tmp_path):
    """The bench's multi-GPU frame path (interleaved 16x16 tiles, chunked trace + NCCL gather to
    rank 0, shard.assemble) with every shard traced, assembled into the image and compared with
    the oracle pixel by pixel. The pool exposes one GPU, so the ranks run one after another in a
    one-rank NCCL group per shard world (bench.FrameStep with --force-dist semantics)."""
    import os
    import subprocess
    import sys
    vol, rays, perm, ref = _frame("cfg5")
    np.save(tmp_path / "ref_xyz.npy", ref["xyz"])
    np.save(tmp_path / "ref_t.npy", ref["t"])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "frame_worker.py"), str(tmp_path)],
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "FRAME OK" in r.stdout


def test_cfg4_street_view_full_frame():
    """SURVEY §8(d) cfg4 "plus a street-level view": eye 40 voxels above the street, looking along
    it (long grazing rays between the buildings), 960x540, every ray vs the oracle."""
    import torch
    import bench
    from inputs import rays as R
    vol = bench.make_volume("city")
    rays, _ = R.camera("city_street", scale=2)
    g = oracle.Grid.from_generator(vol)
    ref = g.trace(rays)
    g.close()
    rt = torch.from_numpy(rays).cuda()
    hits = torch.empty((len(rays), 4), dtype=torch.int32, device="cuda")
    for fmt, h in _handles(vol, ["R(4, 4, 4) G(7)", "G(11)", "S(11)", "T(2, 4) R(3, 3, 3)", "D(4, 4, 4, 6) G(7)"]):
        for restart in (False, True):
            for launch in range(2):
                h.trace(rt, hits, restart=restart, schedule=True)
                out = hits.cpu().numpy()
                assert_parity(out[:, :3], out[:, 3].view(np.float32), ref,
                              f"street {fmt} restart={restart} launch {launch}")
