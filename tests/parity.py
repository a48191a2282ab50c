"""Parity helpers: run the CUDA path (through the C ABI) and the oracle on the same seeded inputs.

Bar (north_star; SURVEY.md §8(c) c-3 row "t"): hit voxel (x,y,z) and the miss flag bit-exact,
|t_gpu - t_ref| <= 1e-4 * max(|t_ref|, 1).
"""
from __future__ import annotations

import numpy as np

T_RTOL = 1e-4


def gpu_trace(handle, rays_np, restart=False, persistent=False):
    import torch
    r = torch.from_numpy(np.ascontiguousarray(rays_np, dtype=np.float32)).cuda()
    h = handle.trace(r, restart=restart, persistent=persistent)
    torch.cuda.synchronize()
    out = h.cpu().numpy()
    xyz = out[:, :3].astype(np.int32)
    t = out[:, 3].view(np.float32)
    return xyz, t


def compare(gpu_xyz, gpu_t, ref, label="", max_report=8):
    """Return (n_mismatch, report string)."""
    rx, rt = ref["xyz"], ref["t"]
    bad_xyz = np.any(gpu_xyz != rx, axis=1)
    hit = rx[:, 0] >= 0
    tol = T_RTOL * np.maximum(np.abs(rt), 1.0)
    with np.errstate(invalid="ignore"):
        bad_t = hit & ~(np.abs(gpu_t.astype(np.float64) - rt.astype(np.float64)) <= tol)
    bad_t |= (~hit) & ~np.isinf(gpu_t)
    bad = bad_xyz | bad_t
    n = int(bad.sum())
    lines = []
    if n:
        idx = np.nonzero(bad)[0][:max_report]
        for i in idx:
            lines.append(f"  ray {i}: gpu {tuple(gpu_xyz[i])} t={gpu_t[i]!r}  ref {tuple(rx[i])} t={rt[i]!r}")
    return n, f"{label}: {n} mismatches of {len(rx)}\n" + "\n".join(lines)


def assert_parity(gpu_xyz, gpu_t, ref, label=""):
    n, rep = compare(gpu_xyz, gpu_t, ref, label)
    assert n == 0, rep
