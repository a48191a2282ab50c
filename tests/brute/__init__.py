"""ctypes loader for tests/brute/brute.c (exact brute-force first hit; a test pin for the oracle)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libbrute.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(HERE, "brute.c")
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", LIB, src])
        L = ctypes.CDLL(LIB)
        vp = ctypes.c_void_p
        L.brute_trace.argtypes = [vp, vp, vp, ctypes.c_int64, vp, vp, vp, vp, vp, ctypes.c_int]
        _lib = L
    return _lib


def trace(occ: np.ndarray, rays: np.ndarray):
    """occ: bool/uint8 (Rz, Ry, Rx); rays (n, 8) fp32. Returns dict(xyz, tnum, tden (t = tnum/tden
    * 2^14 exactly), status (0 miss, 1 hit, 2 non-canonical, 3 non-unique minimum), axes)."""
    o = np.ascontiguousarray(occ, dtype=np.uint8)
    Rz, Ry, Rx = o.shape
    dims = np.array([Rx, Ry, Rz], dtype=np.int32)
    r = np.ascontiguousarray(rays, dtype=np.float32).reshape(-1, 8)
    n = len(r)
    xyz = np.empty((n, 3), np.int32)
    tn, td = np.empty(n, np.int64), np.empty(n, np.int64)
    st, ax = np.empty(n, np.uint8), np.empty(n, np.uint8)
    lib().brute_trace(o.ctypes.data, dims.ctypes.data, r.ctypes.data, n, xyz.ctypes.data, tn.ctypes.data,
                      td.ctypes.data, st.ctypes.data, ax.ctypes.data, 0)
    return dict(xyz=xyz, tnum=tn, tden=td, status=st, axes=ax)
