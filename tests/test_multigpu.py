"""World-size-2 CPU (gloo) test of the multi-GPU host logic: interleaved screen-tile sharding,
the one hit-gather collective and the un-permutation on rank 0."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from inputs import rays as R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, width, height, q):
    import torch
    import torch.distributed as dist
    from paper_2410_14128_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    perm = R.tile_order(width, height)
    own = shard.shard(perm, width, rank, world)
    # stand-in for vf_trace: a hit record that encodes the pixel it belongs to
    pix = perm[own]
    hits = torch.from_numpy(np.stack([pix, pix * 3, -pix, pix % 7], 1).astype(np.int32))
    counts = shard.shard_counts(perm, width, world)
    bufs = shard.gather_hits(hits, counts)
    if rank == 0:
        img = shard.assemble(bufs, perm, width, world)
        q.put(img)
    dist.destroy_process_group()


def test_tile_shard_gather_unpermute_gloo():
    width, height, world = 72, 40, 2  # ragged: tiles at the right/bottom edge are partial
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, width, height, q)) for r in range(world)]
    for p in procs:
        p.start()
    img = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    pix = np.arange(width * height)
    np.testing.assert_array_equal(img[:, 0], pix)
    np.testing.assert_array_equal(img[:, 1], pix * 3)
    np.testing.assert_array_equal(img[:, 2], -pix)
    np.testing.assert_array_equal(img[:, 3], pix % 7)


def test_shards_partition_and_balance():
    from paper_2410_14128_b200 import shard
    perm = R.tile_order(1920, 1080)
    for world in (1, 2, 4, 8):
        parts = [shard.shard(perm, 1920, r, world) for r in range(world)]
        allidx = np.sort(np.concatenate(parts))
        np.testing.assert_array_equal(allidx, np.arange(len(perm)))
        sizes = [len(p) for p in parts]
        assert max(sizes) / (sum(sizes) / world) < 1.03  # interleaved tiles: balanced ray counts
        assert sizes == shard.shard_counts(perm, 1920, world)


def test_tile_order_is_a_permutation_with_warp_tiles():
    perm = R.tile_order(64, 48)
    assert sorted(perm.tolist()) == list(range(64 * 48))
    # the first 32 rays form one 8x4 warp tile
    px, py = perm[:32] % 64, perm[:32] // 64
    assert px.max() - px.min() == 7 and py.max() - py.min() == 3


def _worker_chunked(rank, world, port, width, height, k, q):
    import torch
    import torch.distributed as dist
    from paper_2410_14128_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    perm = R.tile_order(width, height)
    own = shard.shard(perm, width, rank, world)
    pix = torch.from_numpy(perm[own].astype(np.int32))
    counts = shard.shard_counts(perm, width, world)
    pipe = shard.ChunkedGather(counts, k, "cpu")
    seen = []

    def trace_chunk(lo, hi, hv):  # stand-in for vf_trace on local rays [lo, hi)
        seen.append((lo, hi))
        p = pix[lo:hi]
        hv.copy_(torch.stack([p, p * 3, -p, p % 7], 1))

    bufs = pipe.run(trace_chunk)
    # the chunks cover exactly the rank's own rays, in order
    assert seen[0][0] == 0 and seen[-1][1] == counts[rank]
    assert all(a[1] == b[0] for a, b in zip(seen, seen[1:]))
    if rank == 0:
        q.put(shard.assemble(bufs, perm, width, world))
    dist.destroy_process_group()


def test_chunked_trace_gather_pipeline_gloo():
    """SURVEY §8(e) Overlap: the trace/gather pipeline over K row chunks of the padded hit buffers
    reassembles the same frame as one gather (ragged shards, K not dividing the rows)."""
    width, height, world, k = 72, 40, 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_chunked, args=(r, world, port, width, height, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    img = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    pix = np.arange(width * height)
    np.testing.assert_array_equal(img[:, 0], pix)
    np.testing.assert_array_equal(img[:, 1], pix * 3)
    np.testing.assert_array_equal(img[:, 2], -pix)
    np.testing.assert_array_equal(img[:, 3], pix % 7)


def test_chunk_bounds_cover_padded_rows():
    from paper_2410_14128_b200 import shard
    for counts, k in (([10, 7], 3), ([5], 8), ([1000, 999, 998], 4)):
        b = shard.chunk_bounds(counts, k)
        assert b[0][0] == 0 and b[-1][1] == max(counts)
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        assert all(hi > lo for lo, hi in b)


def _nccl_worker(port, q):
    import torch
    import torch.distributed as dist
    import inputs
    from paper_2410_14128_b200 import shard, vf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)  # as bench.py does
    d = inputs.menger(128, 4)
    keys, rgba = inputs.voxels_device(d)
    h = vf.build((keys, rgba, (128, 128, 128)), "G(4) R(3^3)")
    rays_np, perm = R.perspective(64, 48, 60.0, (-40.3, 60.7, -70.1), (40.5, 40.5, 40.5))
    rays = torch.from_numpy(rays_np).to(dev)
    ref = h.trace(rays).cpu().numpy()
    counts = shard.shard_counts(perm, 64, 1)
    pipe = shard.ChunkedGather(counts, 3, dev)  # NCCL gather to self, chunk by chunk, async
    bufs = pipe.run(lambda lo, hi, hv: h.trace(rays[lo:hi], hv))
    torch.cuda.synchronize()
    q.put(bool((bufs[0].cpu().numpy() == ref).all()))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_chunked_gather_over_nccl_single_rank():
    """The bench's N>1 pipeline (trace chunk k, async NCCL gather of chunk k) run for real over NCCL
    with one rank on the box's GPU: the gathered hits equal one whole-frame trace."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    ok = q.get(timeout=300)
    p.join(60)
    assert p.exitcode == 0 and ok


def _bench_frame_worker(rank, world, port, q):
    """bench.py's N > 1 step on CPU/gloo: FrameStep (chunked trace of this rank's interleaved
    tiles + async gather to rank 0) with a stand-in tracer, bench.max_over_ranks, assembly."""
    import sys
    import torch
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_2410_14128_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    width, height = 200, 120  # ragged last tile row/column
    perm = R.tile_order(width, height)
    own = shard.shard(perm, width, rank, world)
    counts = shard.shard_counts(perm, width, world)
    # "rays": the pixel index of each ray; the stand-in trace writes a record derived from it
    rays = torch.from_numpy(perm[own].astype(np.int32))

    def trace(rv, hv):
        hv[:, 0] = rv
        hv[:, 1] = rv * 3
        hv[:, 2] = -rv
        hv[:, 3] = rv % 7

    step = bench.FrameStep(trace, rays, counts, rank, world, True, torch.device("cpu"), chunks=3, timed=False)
    got = step()
    mx = bench.max_over_ranks([float(rank + 1), 10.0 - rank], torch.device("cpu"), True)
    if rank == 0:
        img = shard.assemble(got, perm, width, world)
        q.put((img, mx, step.launches))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_frame_step_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_frame_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    img, mx, launches = q.get(timeout=180)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    pix = np.arange(200 * 120)
    np.testing.assert_array_equal(img[:, 0], pix)
    np.testing.assert_array_equal(img[:, 1], pix * 3)
    np.testing.assert_array_equal(img[:, 2], -pix)
    np.testing.assert_array_equal(img[:, 3], pix % 7)
    assert mx == [2.0, 10.0] and launches == 3


@pytest.mark.gpu
def test_p2p_fused_gather_two_processes(tmp_path):
    """The fused trace + gather over peer memory (vf_trace_scatter into rank 0's frame, mapped by
    CUDA IPC; shard.PeerFrame) with two real processes. The pool exposes one GPU, so both ranks
    run on it: the IPC export / open / scatter path is the one NVLink peers take (cross-process
    mapping, remote stores from the trace kernel). The assembled frame — row-major pixels, no
    un-permutation — must equal the oracle's first hits pixel by pixel (cfg2, 1024x1024)."""
    import subprocess
    import sys
    import oracle
    import bench
    from parity import assert_parity
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    out = str(tmp_path / "frame.npy")
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(root, "tests", "p2p_worker.py"), "cfg2", out],
                                      env=env, cwd=root, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(l[-3000:] for l in logs)
    frame = np.load(out)
    rays, perm = bench.make_rays("cfg2")
    g = oracle.Grid.from_generator(bench.make_volume("menger"))
    ref = g.trace(rays)
    g.close()
    got = frame[perm]  # pixel order -> ray order
    assert_parity(got[:, :3], got[:, 3].view(np.float32), ref, "cfg2 p2p two-process frame")


def _peer_worker(rank, world, port, fail_rank, q):
    import torch
    import torch.distributed as dist
    from paper_2410_14128_b200 import shard
    import paper_2410_14128_b200.vf as vfm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the CUDA IPC calls are stubbed: this checks PeerFrame's host protocol (export on rank 0,
    # broadcast, open elsewhere, every rank agreeing on failure), not the mapping itself
    vfm.ipc_export = lambda t: b"H" * 72
    def _open(blob, dev):
        if rank == fail_rank:
            raise RuntimeError("no peer access")
        assert blob == b"H" * 72
        return 0x1000 + rank
    vfm.ipc_open = _open
    vfm.ipc_close = lambda p: None
    try:
        pf = shard.PeerFrame(10, np.arange(3) + rank, torch.device("cpu"))
        res = ("ok", pf.ptr if rank else -1, pf.slots.tolist(), pf.frame is not None)
    except RuntimeError as e:
        res = ("failed", str(e))
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [None, 1])
def test_peer_frame_protocol_gloo(fail_rank):
    """shard.PeerFrame's host protocol at world size 2 over gloo: rank 0 exports its frame buffer,
    the handle is broadcast, rank 1 maps it; if the mapping fails on any rank, EVERY rank raises
    (so bench.py's FrameStep falls back to the NCCL gather together)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, fail_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    if fail_rank is None:
        assert got[0] == ("ok", -1, [0, 1, 2], True)
        assert got[1] == ("ok", 0x1001, [1, 2, 3], False)
    else:
        assert all(r[0] == "failed" and "no peer access" in r[1] for r in got.values()), got


def _replica_worker(rank, world, port, differ, q):
    import torch.distributed as dist
    from paper_2410_14128_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = {"bytes_used": 1000, "nonempty_voxels": 10, "buffer_checksum": 12345, "query_checksum": 678,
         "query_samples": 64}
    if differ and rank == 1:
        d["buffer_checksum"] += 1
    try:
        q.put((rank, ("ok", shard.verify_replicas(d))))
    except RuntimeError as e:
        q.put((rank, ("differ", str(e))))
    dist.destroy_process_group()


@pytest.mark.parametrize("differ", [False, True])
def test_replica_verification_gloo(differ):
    """SURVEY §8(e) "Replicas": the ranks' volume digests are compared over gloo; a mismatch on any
    rank raises on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, world, port, differ, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    if differ:
        assert all(v[0] == "differ" and "replicas differ" in v[1] for v in got.values()), got
    else:
        assert got == {0: ("ok", 2), 1: ("ok", 2)}


@pytest.mark.gpu
def test_replica_digest_is_deterministic_and_discriminating():
    """Two builds of the same volume and format have equal digests (the replicas of a multi-GPU run);
    a different volume does not."""
    import inputs
    from paper_2410_14128_b200 import shard, vf
    d1, d2 = inputs.menger(128, 4), inputs.menger(128, 3)
    digests = []
    for d in (d1, d1, d2):
        keys, rgba = inputs.voxels_device(d)
        h = vf.build((keys, rgba, (128, 128, 128)), "R(3, 3, 3) G(4)")
        digests.append(shard.replica_digest(h, slabs=4, step=4))
        h.close()
    assert digests[0] == digests[1]
    assert digests[0]["query_checksum"] != digests[2]["query_checksum"]
    assert digests[0]["buffer_checksum"] != digests[2]["buffer_checksum"]
    assert digests[0]["query_samples"] == 4 * 32 * 32
