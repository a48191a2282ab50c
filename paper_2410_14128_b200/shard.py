"""Screen-tile sharding of a frame across ranks and the one collective (hit gather).

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


def assemble(bufs, perm: np.ndarray, width: int, world: int, tile: int = TILE) -> np.ndarray:
    """Un-permute gathered per-rank hits into a row-major (n_pixels, 4) image buffer."""
    n = len(perm)
    out = np.empty((n, 4), dtype=np.int32)
    for r, b in enumerate(bufs):
        idx = shard(perm, width, r, world, tile)
        out[perm[idx]] = b.cpu().numpy() if hasattr(b, "cpu") else b
    return out
