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


def assemble(bufs, perm: np.ndarray, width: int, world: int, tile: int = TILE) -> np.ndarray:
    """Un-permute gathered per-rank hits into a row-major (n_pixels, 4) image buffer."""
    n = len(perm)
    out = np.empty((n, 4), dtype=np.int32)
    for r, b in enumerate(bufs):
        idx = shard(perm, width, r, world, tile)
        out[perm[idx]] = b.cpu().numpy() if hasattr(b, "cpu") else b
    return out
