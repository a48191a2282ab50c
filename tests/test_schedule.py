"""VF_TRACE_SCHEDULE (include/vf.h): the longest-first block order only changes the order in which
128-ray blocks run, so every scheduled launch must equal the oracle ray for ray — on the first
launch (index order), on later launches (order from the previous launch's block durations), with a
ragged last block, across several ray arrays on one handle (one schedule entry each, LRU beyond
32), across streams, and replayed inside a CUDA graph.
"""
from __future__ import annotations

import numpy as np
import pytest

import inputs
import oracle
from inputs import rays as R
from parity import assert_parity

pytestmark = pytest.mark.gpu


def _setup(n_extra=77):
    """~484k rays (3,780 blocks of 128): more than two waves of resident blocks on a B200 (148 SMs x
    8-9 blocks), below which the library does not reorder."""
    import torch
    from paper_2410_14128_b200 import vf
    d = inputs.menger(128, 4)
    keys, rgba = inputs.voxels_device(d)
    h = vf.build((keys, rgba, (128, 128, 128)), "R(3, 3, 3) G(4)")
    rays, _ = R.perspective(800, 600, 60.0, (-40.3, 60.7, -70.1), (40.5, 40.5, 40.5))
    rays = np.concatenate([rays, R.adversarial_rays(4096 + n_extra, (128,) * 3, 3)])  # ragged last block
    ref = oracle.Grid.from_generator(d).trace(rays)
    return torch, vf, h, rays, ref


def test_schedule_state_allocated_only_for_multi_wave_launches():
    """A scheduled launch of > 2 waves allocates the array's schedule (8 B per block, through the
    build's allocator = torch's caching allocator); a one-wave launch does not (index order)."""
    torch, vf, h, rays, ref = _setup()
    small = torch.from_numpy(rays[:20000]).cuda()
    big = torch.from_numpy(rays).cuda()
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_allocated()
    hs = h.trace(small, schedule=True)
    torch.cuda.synchronize()
    m1 = torch.cuda.memory_allocated()
    assert m1 - m0 == hs.numel() * 4, "one-wave launch must not allocate schedule state"
    hb = h.trace(big, schedule=True)
    torch.cuda.synchronize()
    m2 = torch.cuda.memory_allocated()
    nb = (rays.shape[0] + 127) // 128
    need = hb.numel() * 4 + 8 * nb + 8 * rays.shape[0]  # hits + per-block and per-ray schedule state
    assert m2 - m1 >= need, (m2 - m1, need)
    _check(torch, hb, ref, "first scheduled launch")
    h.close()


def _check(torch, hits, ref, label):
    torch.cuda.synchronize()
    o = hits.cpu().numpy()
    assert_parity(o[:, :3], o[:, 3].view(np.float32), ref, label)


@pytest.mark.parametrize("mode", [True, "regroup"])
def test_scheduled_launches_equal_oracle(mode):
    """Block order (and with VF_TRACE_REGROUP the rays regrouped into warps inside 256-ray groups,
    incl. the ragged last group) from the previous launch: every launch equals the oracle."""
    torch, vf, h, rays, ref = _setup()
    rt = torch.from_numpy(rays).cuda()
    for restart in (False, True):
        for it in range(8):  # launch 0: index order; then ordered (regroup: both modes measured)
            hits = h.trace(rt, restart=restart, schedule=mode)
            _check(torch, hits, ref, f"schedule={mode} launch {it} restart={restart}")
            # (regrouping is measured: a launch regroups or not, 4 or 3 kernels)
            assert h.launch_count(rt, restart=restart, schedule=mode) in ((3, 4) if mode == "regroup" else (3,))
    h.close()


def test_schedule_many_arrays_and_streams():
    torch, vf, h, rays, ref = _setup(5)
    # 40 distinct ray arrays (more than the 32 schedule entries: LRU eviction), each traced twice
    arrs = [torch.from_numpy(rays).cuda() for _ in range(40)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for rep in range(2):
        for i, a in enumerate(arrs):
            s = s1 if (i + rep) % 2 else s2
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs.append(h.trace(a, restart=False, schedule=True, stream=s))
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        _check(torch, o, ref, f"array {k % 40} pass {k // 40}")
    h.close()


def test_schedule_inside_cuda_graph():
    torch, vf, h, rays, ref = _setup(31)
    rt = torch.from_numpy(rays).cuda()
    hits = torch.empty((rays.shape[0], 4), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # warm-up outside capture creates the array's schedule entry
            h.trace(rt, hits, schedule=True, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.trace(rt, hits, schedule="regroup", stream=torch.cuda.current_stream())
    for it in range(3):
        hits.zero_()
        g.replay()
        _check(torch, hits, ref, f"graph replay {it}")
    # 34 more arrays push every other entry out (LRU over 32); the captured array's entry is pinned
    others = [rt.clone() for _ in range(34)]
    for o in others:
        for _ in range(2):
            h.trace(o, schedule=True)
    torch.cuda.synchronize()
    del others
    hits.zero_()
    g.replay()
    _check(torch, hits, ref, "graph replay after LRU pressure")
    # an array first seen during capture runs unscheduled (nothing is allocated during capture)
    rt2 = rt.clone()
    hits2 = torch.empty_like(hits)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        h.trace(rt2, hits2, schedule=True, stream=torch.cuda.current_stream())
    g2.replay()
    _check(torch, hits2, ref, "graph, array first seen in capture")
    del g, g2
    h.close()


def test_schedule_scatter_and_host_paths():
    torch, vf, h, rays, ref = _setup(13)
    n = rays.shape[0]
    rt = torch.from_numpy(rays).cuda()
    slots = torch.from_numpy(np.random.default_rng(7).permutation(n).astype(np.int32)).cuda()
    frame = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    for it in range(3):
        frame.zero_()
        h.trace_scatter(rt, frame, slots, schedule=True)
        torch.cuda.synchronize()
        got = frame.cpu().numpy()[slots.cpu().numpy()]
        assert_parity(got[:, :3], got[:, 3].view(np.float32), ref, f"scatter schedule {it}")
    hr = torch.from_numpy(rays).pin_memory()
    hh = torch.empty((n, 4), dtype=torch.int32).pin_memory()
    for it in range(3):
        h.trace_host(hr, hh, schedule=True)
        o = hh.numpy()
        assert_parity(o[:, :3], o[:, 3].view(np.float32), ref, f"host schedule {it}")
    h.close()
