"""Screen-tile sharding of a frame across ranks and the one collective (hit gather): NCCL
(ChunkedGather) or the fused trace + peer-memory scatter (PeerFrame).

north_star / SURVEY.md §8(e): the volume is replicated on every GPU, the frame's rays are
sharded by screen tiles, and NCCL is used only for the final hit-buffer gather. Tiles are
interleaved (`tile mod N`) to balance sky vs geometry (SURVEY E-h: max/mean 1.01-1.03 at N=8).
The helpers are backend-agnostic (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

TILE = 16


def tile_of(perm: np.ndarray, width: int, tile: int = TILE) -> np.ndarray:
    """Screen-tile id of every ray; `perm[i]` is ray i's row-major pixel index."""
    px, py = perm % width, perm // width
    return (py // tile) * ((width + tile - 1) // tile) + (px // tile)


def shard(perm: np.ndarray, width: int, rank: int, world: int, tile: int = TILE) -> np.ndarray:
    """Indices (into the ray array) owned by `rank`: its interleaved tiles, in ray order."""
    return np.nonzero(tile_of(perm, width, tile) % world == rank)[0]


def shard_counts(perm: np.ndarray, width: int, world: int, tile: int = TILE):
    t = tile_of(perm, width, tile) % world
    return [int((t == r).sum()) for r in range(world)]


def replica_digest(handle, slabs: int = 8, step: int = 16) -> dict:
    """Digest of this rank's replica of the volume (SURVEY.md §8(e) "Replicas": every rank builds the
    format from the same descriptor and seed; the build is deterministic): bytes_used, the
    non-empty voxel count, a position-weighted checksum of the format buffer's words, and a
    checksum of vf_query over `slabs` z-slabs sampled every `step` voxels in x and y (the voxels
    the format answers for, through the library's own lookup). Host integers only."""
    import torch
    st = handle.stats()
    words = handle.buffer_words().astype(np.uint64)
    wsum = int(np.sum(words * (2 * np.arange(words.size, dtype=np.uint64) + 1), dtype=np.uint64))
    rx, ry, rz = st["dims"]
    xs, ys = np.arange(0, rx, step), np.arange(0, ry, step)
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    qsum = 0
    for k in range(slabs):
        z = (2 * k + 1) * rz // (2 * slabs)
        xyz = np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, z)], 1).astype(np.int32)
        rgba = handle.query(torch.from_numpy(xyz).cuda()).cpu().numpy().astype(np.uint32).astype(np.uint64)
        qsum = (qsum * 1000003 + int(np.sum(rgba * (2 * np.arange(rgba.size, dtype=np.uint64) + 1),
                                            dtype=np.uint64))) % (1 << 64)
    return {"bytes_used": int(st["bytes_used"]), "nonempty_voxels": int(st["nonempty_voxels"]),
            "buffer_checksum": wsum, "query_checksum": qsum, "query_samples": int(slabs * gx.size)}


def verify_replicas(digest: dict, group=None) -> int:
    """Compare every rank's replica_digest over `group` (a gloo group: host objects, no NCCL);
    raises on every rank if any two differ. Returns the number of ranks compared."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    got = [None] * world
    dist.all_gather_object(got, digest, group=group)
    bad = [r for r, d in enumerate(got) if d != got[0]]
    if bad:
        raise RuntimeError(f"volume replicas differ: rank 0 {got[0]} vs rank(s) {bad}: {[got[r] for r in bad]}")
    return world


def gather_hits(hits, counts, group=None, dst: int = 0):
    """Gather every rank's (n_r, 4) int32 hit buffer to `dst` (one collective). Returns the list
    of per-rank buffers on dst, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    m = max(counts)
    if hits.shape[0] < m:  # collectives move equal-sized buffers: pad ragged shards
        pad = torch.empty((m, hits.shape[1]), dtype=hits.dtype, device=hits.device)
        pad[: hits.shape[0]] = hits
        hits = pad
    if rank == dst:
        bufs = [torch.empty((m, 4), dtype=hits.dtype, device=hits.device) for _ in counts]
        dist.gather(hits, gather_list=bufs, dst=dst, group=group)
        return [b[:c] for b, c in zip(bufs, counts)]
    dist.gather(hits, dst=dst, group=group)
    return None


def chunk_bounds(counts, k: int):
    """Row ranges [lo, hi) of the K gather chunks over the padded (max(counts), 4) hit buffer; the
    same on every rank, so every chunk is one equal-sized collective (SURVEY.md §8(e) Overlap)."""
    m = max(counts)
    k = max(1, min(k, m))
    return [(i * m // k, (i + 1) * m // k) for i in range(k)]


class ChunkedGather:
    """Trace-and-gather pipeline of one frame (SURVEY.md §8(e) "Overlap"): the rank's hit buffer is
    padded to max(counts) rows and cut into K row chunks; after chunk k is traced, its gather to
    `dst` is enqueued asynchronously (the NCCL stream waits only for the work issued so far), so
    chunk k's transfer overlaps the trace of chunk k+1. Still exactly one kind of collective: a
    gather of hit records to rank 0."""

    def __init__(self, counts, k: int, device, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist
        self.counts, self.group, self.dst = counts, group, dst
        self.rank = dist.get_rank(group)
        self.m = max(counts)
        self.bounds = chunk_bounds(counts, k)
        self.hits = torch.empty((self.m, 4), dtype=torch.int32, device=device)
        self.recv = ([torch.empty((self.m, 4), dtype=torch.int32, device=device) for _ in counts]
                     if self.rank == dst else None)

    def run(self, trace_chunk):
        """trace_chunk(lo, hi, hits_view) traces local rays [lo, hi) into hits_view; rows beyond the
        rank's count are padding. Returns the list of per-rank hit buffers on dst, None elsewhere."""
        import torch.distributed as dist
        n_local = self.counts[self.rank]
        works = []
        for lo, hi in self.bounds:
            hl = min(hi, n_local)
            if hl > lo:
                trace_chunk(lo, hl, self.hits[lo:hl])
            gl = [b[lo:hi] for b in self.recv] if self.recv is not None else None
            works.append(dist.gather(self.hits[lo:hi], gather_list=gl, dst=self.dst, group=self.group,
                                     async_op=True))
        for w in works:
            w.wait()
        if self.recv is None:
            return None
        return [b[:c] for b, c in zip(self.recv, self.counts)]


class PeerFrame:
    """The fused trace + gather of one frame over peer memory (the task's "compute
    step followed by a collective in ONE kernel"): rank 0 owns the frame's hit buffer in
    row-major pixel order; every rank maps it (CUDA IPC, vf_ipc_open: NVLink / NVSwitch between
    GPUs of one node) and traces its interleaved tiles with vf_trace_scatter, whose kernel stores
    each hit straight into rank 0's image at the ray's pixel. A one-int all-reduce after the trace
    is the completion signal (stream-ordered after every rank's kernel). No hit gather, no
    un-permutation. Raises on any rank if the mapping fails on any rank (the caller falls back to
    ChunkedGather)."""

    def __init__(self, n_total: int, pixels_local: np.ndarray, device, group=None):
        import torch
        import torch.distributed as dist
        from paper_2410_14128_b200 import vf
        self.rank, self.group = dist.get_rank(group), group
        self.device = device
        self.frame = torch.empty((n_total, 4), dtype=torch.int32, device=device) if self.rank == 0 else None
        blob = [vf.ipc_export(self.frame) if self.rank == 0 else None]
        dist.broadcast_object_list(blob, src=0, group=group)
        err = ""
        self.ptr, self._opened = 0, False
        if self.rank == 0:
            self.ptr = self.frame.data_ptr()
        else:
            try:
                self.ptr = vf.ipc_open(blob[0], device.index)
                self._opened = True
            except Exception as e:  # reported to every rank below
                err = str(e)
        errs = [None] * dist.get_world_size(group)
        dist.all_gather_object(errs, err, group=group)
        if any(errs):
            self.close()
            raise RuntimeError("peer frame mapping failed: " + "; ".join(e for e in errs if e))
        self.slots = torch.from_numpy(np.ascontiguousarray(pixels_local, dtype=np.int32)).to(device)
        self.flag = torch.ones(1, dtype=torch.int32, device=device)

    def run(self, trace_scatter, rays):
        """trace_scatter(rays, dest_ptr, slots) traces this rank's rays into the shared frame; then the
        completion signal. Returns the frame on rank 0 (row-major pixels), None elsewhere."""
        import torch.distributed as dist
        trace_scatter(rays, self.ptr, self.slots)
        dist.all_reduce(self.flag, group=self.group)
        return self.frame

    def close(self):
        from paper_2410_14128_b200 import vf
        if self._opened:
            vf.ipc_close(self.ptr)
            self._opened = False


def assemble(bufs, perm: np.ndarray, width: int, world: int, tile: int = TILE) -> np.ndarray:
    """Un-permute gathered per-rank hits into a row-major (n_pixels, 4) image buffer."""
    n = len(perm)
    out = np.empty((n, 4), dtype=np.int32)
    for r, b in enumerate(bufs):
        idx = shard(perm, width, r, world, tile)
        out[perm[idx]] = b.cpu().numpy() if hasattr(b, "cpu") else b
    return out
