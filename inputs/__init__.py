"""inputs — seeded synthetic inputs shared by the oracle and the product path.

INPUT DEFINITION ONLY (task rule ③): volume generators (volgen.h, materialised by
libvolgen.so) and ray generators (rays.py). No ray traversal, DDA or format code here.

Volume presets follow SURVEY.md §8(d) (cfg1..cfg5), the procedural analogues of the
paper's voxelised meshes (§6 "San Miguel, Hairball, Buddha, and Sponza").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvolgen.so")

VG_EMPTY, VG_SPHERE, VG_MENGER, VG_TERRAIN, VG_CITY, VG_SPARSE, VG_RANDOM, VG_BOX, VG_SINGLE, VG_SOLID = range(10)


class VgDesc(ctypes.Structure):
    _fields_ = [("gen", ctypes.c_uint32), ("dims", ctypes.c_uint32 * 3), ("seed", ctypes.c_uint32),
                ("tex", ctypes.c_uint32), ("p", ctypes.c_int32 * 8)]


def desc(gen: int, dims, seed: int = 0, tex: int = 0, params=()) -> VgDesc:
    d = VgDesc()
    d.gen = gen
    if isinstance(dims, int):
        dims = (dims, dims, dims)
    for a in range(3):
        d.dims[a] = int(dims[a])
    d.seed = seed & 0xFFFFFFFF
    d.tex = tex
    for i, v in enumerate(params):
        d.p[i] = int(v) if int(v) < 2**31 else int(v) - 2**32
    return d


def dims_of(d: VgDesc):
    return (int(d.dims[0]), int(d.dims[1]), int(d.dims[2]))


# ---- presets -------------------------------------------------------
def sphere(R: int = 64, r: int = 28) -> VgDesc:          # G1, cfg1
    return desc(VG_SPHERE, R, params=(r,))


def menger(R: int = 256, k: int = 5) -> VgDesc:           # G2, cfg2
    return desc(VG_MENGER, R, params=(k,))


def terrain(R: int = 1024, seed: int = 0x24101412) -> VgDesc:   # G3, cfg3
    return desc(VG_TERRAIN, R, seed=seed)


def city(R: int = 2048, seed: int = 0x0C17, tex: int = 1) -> VgDesc:  # G4, cfg4
    return desc(VG_CITY, R, seed=seed, tex=tex)


def sparse(R: int = 4096, seed: int = 0x4096) -> VgDesc:   # G5, cfg5
    return desc(VG_SPARSE, R, seed=seed)


def random_occupancy(dims, p: float, seed: int) -> VgDesc:
    return desc(VG_RANDOM, dims, seed=seed, params=(min(int(p * 2**32), 2**32 - 1),))


def box(dims, lo, hi) -> VgDesc:
    return desc(VG_BOX, dims, params=tuple(lo) + tuple(hi))


def single(dims, xyz) -> VgDesc:
    return desc(VG_SINGLE, dims, params=tuple(xyz))


def solid(dims) -> VgDesc:
    return desc(VG_SOLID, dims)


def empty(dims) -> VgDesc:
    return desc(VG_EMPTY, dims)


# ---- native library ------------------------------------------------------------------------
def build(force: bool = False) -> str:
    src = os.path.join(HERE, "volgen_lib.cu")
    hdr = os.path.join(HERE, "volgen.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    cmd = ["nvcc", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-o", LIB_PATH, src]
    subprocess.check_call(cmd, cwd=HERE)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER(VgDesc)
        L.vg_dense_host.argtypes = [P, ctypes.c_void_p]
        L.vg_dense_host.restype = ctypes.c_int
        L.vg_voxels_host.argtypes = [P, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.vg_voxels_host.restype = ctypes.c_int
        L.vg_sparse_objects.argtypes = [ctypes.c_uint32, ctypes.c_void_p]
        L.vg_voxel_host.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.vg_voxel_host.restype = ctypes.c_uint32
        L.vg_count_device.argtypes = [P, ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p]
        L.vg_count_device.restype = ctypes.c_int
        L.vg_extract_device.argtypes = [P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p]
        L.vg_extract_device.restype = ctypes.c_int
        L.vg_dense_device.argtypes = [P, ctypes.c_void_p, ctypes.c_void_p]
        L.vg_dense_device.restype = ctypes.c_int
        _lib = L
    return _lib


def dense_host(d: VgDesc) -> np.ndarray:
    """Dense x-fastest RGBA volume as a numpy array of shape (Rz, Ry, Rx), uint32."""
    Rx, Ry, Rz = dims_of(d)
    out = np.zeros((Rz, Ry, Rx), dtype=np.uint32)
    rc = lib().vg_dense_host(ctypes.byref(d), out.ctypes.data)
    assert rc == 0
    return out


def voxel_host(d: VgDesc, x: int, y: int, z: int) -> int:
    return int(lib().vg_voxel_host(ctypes.byref(d), x, y, z))


def voxels_host(d: VgDesc, xyz: np.ndarray) -> np.ndarray:
    """Voxel words at the points xyz ((n, 3) int64; outside the volume -> 0)."""
    p = np.ascontiguousarray(xyz, dtype=np.int64).reshape(-1, 3)
    out = np.empty(len(p), dtype=np.uint32)
    assert lib().vg_voxels_host(ctypes.byref(d), p.ctypes.data, len(p), out.ctypes.data) == 0
    return out


def sparse_objects(seed: int = 0x4096) -> np.ndarray:
    """G5 object table (4096, 6) int32: cx, cy, cz, r, box, col."""
    out = np.empty((4096, 6), dtype=np.int32)
    lib().vg_sparse_objects(seed & 0xFFFFFFFF, out.ctypes.data)
    return out


def voxels_device(d: VgDesc, stream=None):
    """Non-empty voxels on the current CUDA device: (keys int64 x|y<<21|z<<42, rgba int32)."""
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    n = ctypes.c_uint64(0)
    rc = lib().vg_count_device(ctypes.byref(d), ctypes.byref(n), ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"vg_count_device failed: cuda error {rc}")
    cap = max(int(n.value), 1)
    keys = torch.empty(cap, dtype=torch.int64, device="cuda")
    rgba = torch.empty(cap, dtype=torch.int32, device="cuda")
    m = ctypes.c_uint64(0)
    rc = lib().vg_extract_device(ctypes.byref(d), ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(rgba.data_ptr()),
                                 cap, ctypes.byref(m), ctypes.c_void_p(s.cuda_stream))
    if rc != 0 or m.value != n.value:
        raise RuntimeError(f"vg_extract_device failed: rc={rc} n={n.value} m={m.value}")
    return keys[: n.value], rgba[: n.value]


def dense_device(d: VgDesc, stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    Rx, Ry, Rz = dims_of(d)
    out = torch.empty((Rz, Ry, Rx), dtype=torch.int32, device="cuda")
    rc = lib().vg_dense_device(ctypes.byref(d), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"vg_dense_device failed: cuda error {rc}")
    return out
