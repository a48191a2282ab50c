"""Exact brute-force first hit with Python Fractions — the oracle's independent pin.

SURVEY.md §8(c) c-1 "Equivalent brute-force form": voxel v is pierced iff
max(t_start, t_enter(v)) < min(t_end, t_exit(v)) (strictly positive length), with
half-open membership on zero-direction axes; the result is the pierced non-empty v with
minimum entry time, which is unique. Shares nothing with oracle/oracle.c: rational
arithmetic is Python's ``fractions.Fraction`` (exact for every fp32 input), there is no
walk, no plane ordering and no integer scaling.

Per axis a, the set of t with cell index v_a (right-limit semantics, reading A2):
  d_a > 0: v_a <= o_a + t d_a <  v_a + 1   -> t in [(v_a - o_a)/d_a, (v_a + 1 - o_a)/d_a)
  d_a < 0: v_a <  o_a + t d_a <= v_a + 1   -> t in [(v_a + 1 - o_a)/d_a, (v_a - o_a)/d_a)
  d_a = 0: all t if floor(o_a) == v_a, else none.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def first_hit(occ: np.ndarray, ray) -> tuple:
    """occ: boolean (Rz, Ry, Rx). ray: 8 floats. Returns (x, y, z, t_exact Fraction) or None."""
    Rz, Ry, Rx = occ.shape
    R = (Rx, Ry, Rz)
    o = [Fraction(float(np.float32(ray[i]))) for i in range(3)]
    d = [Fraction(float(np.float32(ray[4 + i]))) for i in range(3)]
    tmin = Fraction(float(np.float32(ray[3])))
    tmax_f = float(np.float32(ray[7]))
    tmax = None if math.isinf(tmax_f) else Fraction(tmax_f)
    if all(x == 0 for x in d):
        return None
    # per-axis interval of t for each cell index (None = empty, "all" = whole line)
    iv = []
    for a in range(3):
        if d[a] == 0:
            c = math.floor(o[a])
            iv.append({c: "all"} if 0 <= c < R[a] else {})
            continue
        m = {}
        for v in range(R[a]):
            if d[a] > 0:
                lo, hi = (v - o[a]) / d[a], (v + 1 - o[a]) / d[a]
            else:
                lo, hi = (v + 1 - o[a]) / d[a], (v - o[a]) / d[a]
            m[v] = (lo, hi)
        iv.append(m)
    best = None
    zs, ys, xs = np.nonzero(occ)
    for x, y, z in zip(xs.tolist(), ys.tolist(), zs.tolist()):
        lo, hi = tmin, tmax
        ok = True
        enters = {}
        for a, v in enumerate((x, y, z)):
            e = iv[a].get(v)
            if e is None:
                ok = False
                break
            if e == "all":
                continue
            enters[a] = e[0]
            if e[0] > lo:
                lo = e[0]
            if hi is None or e[1] < hi:
                hi = e[1]
        if not ok:
            continue
        if hi is not None and not (lo < hi):
            continue
        if best is None or lo < best[3]:
            # entry face: axes whose slab is entered exactly at the entry time, unless the
            # segment starts inside the voxel (entry time == tmin)
            axes = [a for a, t in enters.items() if t == lo and lo > tmin]
            best = (x, y, z, lo, axes)
    return best


def trace(occ: np.ndarray, rays: np.ndarray, with_normal: bool = False):
    """Convenience wrapper: (xyz (n,3) int, t_exact list[Fraction|None][, normal (n,3) int8]).
    normal = -sign(d_a) on the lowest entry axis, 0 when starting inside the hit voxel."""
    rays = np.asarray(rays, dtype=np.float32).reshape(-1, 8)
    xyz = np.full((len(rays), 3), -1, dtype=np.int64)
    nrm = np.zeros((len(rays), 3), dtype=np.int8)
    ts = []
    for i, r in enumerate(rays):
        h = first_hit(occ, r)
        if h is None:
            ts.append(None)
        else:
            xyz[i] = h[:3]
            ts.append(h[3])
            if h[4]:
                a = min(h[4])
                nrm[i, a] = -1 if r[4 + a] > 0 else 1
    return (xyz, ts, nrm) if with_normal else (xyz, ts)
