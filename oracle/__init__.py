"""oracle — CPU oracle for first-hit ray intersection. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this package. The product path (paper_2410_14128_b200/) never imports it
and shares no code with it (the one shared module is ``inputs``, the seeded input
generators). See oracle/oracle.c for the definition it implements (SURVEY.md §8(c) c-1/c-2,
PAPER.md:38, :54, :183-185, :203) and tests/brute_force.py for the independent brute-force pin.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

import inputs

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    hdr = os.path.join(os.path.dirname(HERE), "inputs", "volgen.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", LIB_PATH, src], cwd=HERE)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        vp, P = ctypes.c_void_p, ctypes.POINTER(inputs.VgDesc)
        L.oracle_grid_from_dense.argtypes = [vp, ctypes.POINTER(ctypes.c_uint32)]
        L.oracle_grid_from_dense.restype = vp
        L.oracle_grid_from_generator.argtypes = [P, ctypes.c_int]
        L.oracle_grid_from_generator.restype = vp
        L.oracle_grid_procedural.argtypes = [P]
        L.oracle_grid_procedural.restype = vp
        L.oracle_grid_free.argtypes = [vp]
        L.oracle_grid_count.argtypes = [vp]
        L.oracle_grid_count.restype = ctypes.c_uint64
        L.oracle_grid_slab_counts.argtypes = [vp, vp]
        L.oracle_grid_get.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.oracle_grid_get.restype = ctypes.c_int
        L.oracle_grid_get_many.argtypes = [vp, vp, ctypes.c_int64, vp]
        L.oracle_grid_box.argtypes = [vp, vp, vp, vp]
        L.oracle_trace.argtypes = [vp, vp, ctypes.c_int64, vp, vp, vp, vp, vp, ctypes.c_int]
        L.oracle_trace.restype = ctypes.c_int64
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


class Grid:
    """Dense occupancy grid (the uncompressed volume the oracle walks)."""

    def __init__(self, ptr, dims):
        if not ptr:
            raise MemoryError("oracle grid allocation failed")
        self._p = ptr
        self.dims = tuple(int(x) for x in dims)

    @classmethod
    def from_dense(cls, rgba: np.ndarray):
        """rgba: (Rz, Ry, Rx) array, 0 = empty."""
        a = np.ascontiguousarray(rgba, dtype=np.uint32)
        Rz, Ry, Rx = a.shape
        dims = (ctypes.c_uint32 * 3)(Rx, Ry, Rz)
        return cls(lib().oracle_grid_from_dense(a.ctypes.data, dims), (Rx, Ry, Rz))

    @classmethod
    def from_generator(cls, d: "inputs.VgDesc", nthreads: int = 0):
        return cls(lib().oracle_grid_from_generator(ctypes.byref(d), nthreads), inputs.dims_of(d))

    @classmethod
    def procedural(cls, d: "inputs.VgDesc"):
        return cls(lib().oracle_grid_procedural(ctypes.byref(d)), inputs.dims_of(d))

    def count(self) -> int:
        return int(lib().oracle_grid_count(self._p))

    def slab_counts(self) -> np.ndarray:
        out = np.zeros(self.dims[2], dtype=np.uint64)
        lib().oracle_grid_slab_counts(self._p, out.ctypes.data)
        return out

    def get(self, x, y, z) -> int:
        return int(lib().oracle_grid_get(self._p, x, y, z))

    def get_many(self, xyz: np.ndarray) -> np.ndarray:
        """Occupancy (0/1 uint8) at the points xyz ((n, 3) int64, inside the volume)."""
        p = np.ascontiguousarray(xyz, dtype=np.int64).reshape(-1, 3)
        out = np.empty(len(p), dtype=np.uint8)
        lib().oracle_grid_get_many(self._p, p.ctypes.data, len(p), out.ctypes.data)
        return out

    def box(self, lo, ext) -> np.ndarray:
        """Occupancy of the box [lo, lo + ext) as a (ez, ey, ex) uint8 array."""
        lo_ = np.asarray(lo, dtype=np.int64)
        ex_ = np.asarray(ext, dtype=np.int64)
        out = np.empty((int(ex_[2]), int(ex_[1]), int(ex_[0])), dtype=np.uint8)
        lib().oracle_grid_box(self._p, lo_.ctypes.data, ex_.ctypes.data, out.ctypes.data)
        return out

    def trace(self, rays: np.ndarray, nthreads: int = 0, with_steps: bool = False):
        """rays: (n, 8) float32 (vf_ray layout). Returns dict(xyz (n,3) int32, t (n,) float32,
        status (n,) uint8: 0 miss / 1 hit / 2 non-canonical, normal (n,3) int8 entry face,
        steps (n,) int64 optional)."""
        r = np.ascontiguousarray(rays, dtype=np.float32).reshape(-1, 8)
        n = len(r)
        xyz = np.empty((n, 3), dtype=np.int32)
        t = np.empty(n, dtype=np.float32)
        st = np.empty(n, dtype=np.uint8)
        steps = np.empty(n, dtype=np.int64) if with_steps else None
        normal = np.empty((n, 3), dtype=np.int8)
        lib().oracle_trace(self._p, r.ctypes.data, n, xyz.ctypes.data, t.ctypes.data, st.ctypes.data,
                           steps.ctypes.data if steps is not None else None, normal.ctypes.data, nthreads)
        out = dict(xyz=xyz, t=t, status=st, normal=normal)
        if steps is not None:
            out["steps"] = steps
        return out

    def close(self):
        if self._p:
            lib().oracle_grid_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def max_threads() -> int:
    return int(lib().oracle_max_threads())
