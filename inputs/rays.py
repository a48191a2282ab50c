"""inputs/rays.py — seeded ray generators (INPUT DEFINITION ONLY).

Shared by the oracle tests and the GPU product path (task rule ③: the one
module both sides may import). It holds none of the method's arithmetic: it
only produces fp32 ray records ``{ox, oy, oz, tmin, dx, dy, dz, tmax}`` (32 B,
the layout of ``vf_ray`` in include/vf.h) in grid units.

Conventions (SURVEY.md §8(b) "Canonical ray domain", §8(c) A1/A5):
  * grid units: voxel (i,j,k) occupies [i,i+1)x[j,j+1)x[k,k+1);
  * directions need not be normalised; camera directions are normalised in
    fp64, rounded to fp32, then canonicalised;
  * canonical domain: |o_a| in {0} U [2^-16, 2^20), |d_a| in {0} U [2^-30, 2],
    d != 0, 0 <= tmin < tmax, tmin / finite tmax in {0} U [2^-16, 2^20).
    ``canonicalize`` flushes |d_a| < 2^-30 and |o_a| < 2^-16 to +0.
  * camera rays are emitted in screen-tile order: 16x16 pixel blocks, each made
    of 8x4-pixel warp tiles (SURVEY.md §8(d) issue-budget note, E-h); ``perm``
    maps ray index -> pixel index (row-major) so hits can be un-permuted.
"""
from __future__ import annotations

import math

import numpy as np

RAY_DTYPE = np.dtype([("ox", "<f4"), ("oy", "<f4"), ("oz", "<f4"), ("tmin", "<f4"),
                      ("dx", "<f4"), ("dy", "<f4"), ("dz", "<f4"), ("tmax", "<f4")])
assert RAY_DTYPE.itemsize == 32

D_FLUSH = 2.0 ** -30
O_FLUSH = 2.0 ** -16


def pack(o: np.ndarray, d: np.ndarray, tmin=0.0, tmax=np.inf) -> np.ndarray:
    """Pack origins/directions (n,3) into an (n,8) float32 array (vf_ray layout)."""
    o = np.asarray(o, dtype=np.float64).reshape(-1, 3)
    d = np.asarray(d, dtype=np.float64).reshape(-1, 3)
    n = max(len(o), len(d))
    o = np.broadcast_to(o, (n, 3))
    d = np.broadcast_to(d, (n, 3))
    r = np.empty((n, 8), dtype=np.float32)
    r[:, 0:3] = o.astype(np.float32)
    r[:, 4:7] = d.astype(np.float32)
    r[:, 3] = np.broadcast_to(np.asarray(tmin, dtype=np.float64), (n,)).astype(np.float32)
    r[:, 7] = np.broadcast_to(np.asarray(tmax, dtype=np.float64), (n,)).astype(np.float32)
    return canonicalize(r)


def canonicalize(r: np.ndarray) -> np.ndarray:
    """Flush tiny components so every ray lies in the canonical domain (A5)."""
    r = np.array(r, dtype=np.float32, copy=True).reshape(-1, 8)
    d = r[:, 4:7]
    d[np.abs(d) < D_FLUSH] = 0.0
    d[d == 0] = 0.0  # -0 -> +0
    o = r[:, 0:3]
    o[np.abs(o) < O_FLUSH] = 0.0
    o[o == 0] = 0.0
    t = r[:, [3, 7]]
    t[(np.abs(t) < O_FLUSH)] = 0.0
    r[:, [3, 7]] = t
    return r


def tile_order(width: int, height: int, block: int = 16, warp_w: int = 8, warp_h: int = 4) -> np.ndarray:
    """Pixel indices (row-major, y*width+x) in tile order: blocks of block x block pixels,
    each traversed as warp_w x warp_h warp tiles. Partial tiles at the right/bottom
    edge are emitted with only their in-range pixels."""
    ys, xs = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    bx, by = xs // block, ys // block
    lx, ly = xs % block, ys % block
    wx, wy = lx // warp_w, ly // warp_h
    ix, iy = lx % warp_w, ly % warp_h
    nbx = (width + block - 1) // block
    wpr = block // warp_w
    key = ((by * nbx + bx) * (block * block) + (wy * wpr + wx) * (warp_w * warp_h) + iy * warp_w + ix)
    return np.argsort(key.ravel(), kind="stable").astype(np.int64)


def ortho(nx: int, ny: int, spacing: float, z0: float, direction=(0.0, 0.0, 1.0), offset=(0.0, 0.0)):
    """Orthographic rays: origin ((i+.5)*spacing+off_x, (j+.5)*spacing+off_y, z0), fixed direction.
    cfg1: 256x256, spacing 1/4, z0 = -1, d = +z. Returns (rays, perm)."""
    perm = tile_order(nx, ny)
    px, py = perm % nx, perm // nx
    o = np.stack([(px + 0.5) * spacing + offset[0], (py + 0.5) * spacing + offset[1],
                  np.full(px.shape, z0, dtype=np.float64)], axis=1)
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    return pack(o, d[None, :]), perm


def perspective(width: int, height: int, fov_deg: float, eye, target, up=(0.0, 1.0, 0.0)):
    """Pinhole camera through pixel centres; vertical field of view fov_deg.
    Directions normalised in fp64, rounded to fp32, canonicalised. Returns (rays, perm)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    upv = np.cross(right, fwd)
    th = math.tan(math.radians(fov_deg) * 0.5)
    aspect = width / height
    perm = tile_order(width, height)
    px, py = perm % width, perm // width
    sx = ((px + 0.5) / width * 2.0 - 1.0) * th * aspect
    sy = (1.0 - (py + 0.5) / height * 2.0) * th
    d = fwd[None, :] + sx[:, None] * right[None, :] + sy[:, None] * upv[None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return pack(eye[None, :], d), perm


def random_rays(n: int, dims, seed: int, inside_frac: float = 0.3):
    """Random rays aimed at a random point in the volume, from outside or inside the box."""
    rng = np.random.Generator(np.random.MT19937(seed))
    dims = np.asarray(dims, dtype=np.float64)
    tgt = rng.random((n, 3)) * dims
    c = dims / 2
    rad = np.linalg.norm(dims) * 0.75
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    o = c + u * rad * rng.uniform(0.8, 1.6, size=(n, 1))
    inside = rng.random(n) < inside_frac
    o[inside] = rng.random((inside.sum(), 3)) * dims
    d = tgt - o
    d[inside] = rng.normal(size=(inside.sum(), 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return pack(o, d)


def adversarial_rays(n: int, dims, seed: int) -> np.ndarray:
    """Lattice-degenerate rays that hit exact edge/corner ties:
    integer / half-integer origins, directions from {0,+-1,+-2,+-3}^3, axis-parallel rays in
    cell planes, origins on faces/edges/inside the volume, grazing box faces, tmin > 0 starts,
    finite tmax ending exactly on planes."""
    rng = np.random.Generator(np.random.MT19937(seed))
    dims = np.asarray(dims, dtype=np.int64)
    out = []
    kinds = rng.integers(0, 6, size=n)
    for k in kinds:
        if k == 0:  # integer origin outside, small-integer direction
            o = rng.integers(-3, dims + 4).astype(np.float64)
            d = rng.integers(-3, 4, size=3).astype(np.float64)
        elif k == 1:  # half-integer origin anywhere
            o = rng.integers(-2 * 2, 2 * dims + 5) / 2.0
            d = rng.integers(-3, 4, size=3).astype(np.float64)
        elif k == 2:  # axis-parallel, lying in a cell plane
            o = rng.integers(0, dims + 1).astype(np.float64)
            a = rng.integers(0, 3)
            o[a] = -1.5 if rng.random() < 0.5 else dims[a] + 1.5
            d = np.zeros(3)
            d[a] = 1.0 if o[a] < 0 else -1.0
            if rng.random() < 0.5:  # tilt within a plane
                b = (a + 1 + rng.integers(0, 2)) % 3
                d[b] = float(rng.integers(-2, 3))
        elif k == 3:  # origin on a face / edge of the box, direction inward-ish
            o = rng.integers(0, dims + 1).astype(np.float64)
            for a in range(3):
                if rng.random() < 0.5:
                    o[a] = 0.0 if rng.random() < 0.5 else float(dims[a])
            d = rng.integers(-3, 4, size=3).astype(np.float64)
        elif k == 4:  # grazing: origin exactly on the plane of a box face, direction along it
            a = rng.integers(0, 3)
            o = rng.uniform(-2, dims + 2)
            o[a] = 0.0 if rng.random() < 0.5 else float(dims[a])
            d = rng.normal(size=3)
            d[a] = 0.0
            o = np.round(o * 4) / 4
            d = np.round(d * 8) / 8
        else:  # random dyadic origin and direction
            o = np.round(rng.uniform(-3, dims + 3) * 16) / 16
            d = np.round(rng.normal(size=3) * 16) / 16
        if not np.any(d):
            d = np.array([1.0, 1.0, 1.0])
        while np.abs(d).max() > 2.0:  # canonical domain |d_a| <= 2; halving keeps every tie
            d = d * 0.5
        tmin = 0.0
        tmax = np.inf
        r = rng.random()
        if r < 0.2:
            tmin = float(rng.integers(1, 4)) / 2.0
        elif r < 0.3:
            tmax = float(rng.integers(1, 2 * int(dims.max()) + 2)) / 2.0
        out.append((o, d, tmin, tmax))
    o = np.array([x[0] for x in out])
    d = np.array([x[1] for x in out])
    tmin = np.array([x[2] for x in out])
    tmax = np.array([x[3] for x in out])
    return pack(o, d, tmin, tmax)


# ---- workload camera presets -------------------------------------

CAMERAS = {
    # cfg2: 256^3 Menger, 1024^2, fov 60
    "menger": dict(width=1024, height=1024, fov_deg=60.0, eye=(-150.3, 180.7, -210.1),
                   target=(121.5, 121.5, 121.5)),
    "menger_tunnel": dict(width=1024, height=1024, fov_deg=60.0, eye=(121.5, 121.5, -20.25),
                          target=(121.5, 121.5, 121.5)),
    # cfg3: 1024^3 terrain, 1920x1080, fov 70
    "terrain": dict(width=1920, height=1080, fov_deg=70.0, eye=(100.5, 700.25, 90.75),
                    target=(700.0, 350.0, 800.0)),
    # cfg4: 2048^3 city, 1920x1080 aerial, fov 60
    "city": dict(width=1920, height=1080, fov_deg=60.0, eye=(-200.5, 1600.25, -300.75),
                 target=(1024.0, 200.0, 1024.0)),
    "city_street": dict(width=1920, height=1080, fov_deg=60.0, eye=(16.5, 40.25, 8.75),
                        target=(1024.0, 120.0, 1024.0)),
    # Table 2 512^3 rows: 512^3 city, 1024^2 aerial
    "city512": dict(width=1024, height=1024, fov_deg=60.0, eye=(-50.5, 400.25, -75.75),
                    target=(256.0, 50.0, 256.0)),
    # cfg5: 4096^3 sparse, 3840x2160, fov 75, outside one corner
    "sparse": dict(width=3840, height=2160, fov_deg=75.0, eye=(-300.5, -250.25, -350.75),
                   target=(2048.0, 2048.0, 2048.0)),
}


def camera(name: str, scale: int = 1):
    """Rays for a named preset; ``scale`` > 1 subsamples the resolution (for small tests)."""
    c = dict(CAMERAS[name])
    c["width"] //= scale
    c["height"] //= scale
    return perspective(**c)


def incoherent(n: int, lo, hi, seed: int, tmax: float = np.inf):
    """Incoherent secondary-style rays (the regime where memory binds):
    origins uniform in the box [lo, hi), directions uniform on the sphere, segment [0, tmax).
    Adjacent rays share nothing, so a warp's 32 rays touch 32 unrelated paths."""
    rng = np.random.Generator(np.random.MT19937(seed))
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    o = lo + rng.random((n, 3)) * (hi - lo)
    o = np.round(o * 64) / 64 + 1.0 / 128  # dyadic, never exactly on a plane
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return pack(o, d, 0.0, tmax)


def secondary(prim: np.ndarray, xyz: np.ndarray, t: np.ndarray, normal: np.ndarray, seed: int,
              light_dir=(0.35, 1.0, 0.2), ao_tmax: float = 48.0):
    """Shadow + ambient-occlusion rays spawned from primary hits (the
    secondary bounces the paper leaves out). Input only: the primary rays, their hit
    voxels, entry times and entry-face normals (oracle or vf_trace_ex). For every primary ray that
    hit a voxel through a face (normal != 0), in primary-ray order:
      * origin: the hit point o + t d (fp64 from the fp32 values), moved off the entry face into
        the empty neighbour cell: face axis a gets the plane coordinate + 1/64 * normal_a;
      * shadow ray: direction L = normalise(light_dir), mirrored in the face plane if it points
        into the surface; tmax = +inf;
      * AO ray: cosine-weighted direction on the hemisphere around the normal (MT19937(seed)),
        tmax = ao_tmax.
    Returns (n_shadow + n_ao, 8) fp32: all shadow rays first, then all AO rays (each half in the
    primary order, so warps stay screen-coherent), and the primary index of every ray."""
    prim = np.asarray(prim, dtype=np.float32).reshape(-1, 8)
    normal = np.asarray(normal, dtype=np.int64).reshape(-1, 3)
    ok = (np.asarray(xyz)[:, 0] >= 0) & (np.abs(normal).sum(1) == 1)
    src = np.nonzero(ok)[0]
    o = prim[src, 0:3].astype(np.float64)
    d = prim[src, 4:7].astype(np.float64)
    tt = np.asarray(t, dtype=np.float32)[src].astype(np.float64)
    nrm = normal[src].astype(np.float64)
    v = np.asarray(xyz, dtype=np.int64)[src].astype(np.float64)
    p = o + tt[:, None] * d
    face = np.abs(nrm) > 0
    plane = v + (nrm > 0)  # entry face plane on the normal's axis
    p = np.where(face, plane + nrm / 64.0, p)
    L = np.asarray(light_dir, dtype=np.float64)
    L = L / np.linalg.norm(L)
    sd = np.broadcast_to(L, p.shape).copy()
    into = (sd * nrm).sum(1) < 0
    sd[into] = np.where(face[into], -sd[into], sd[into])
    rng = np.random.Generator(np.random.MT19937(seed))
    u1, u2 = rng.random(len(src)), rng.random(len(src))
    r, phi = np.sqrt(u1), 2 * np.pi * u2
    local = np.stack([r * np.cos(phi), r * np.sin(phi), np.sqrt(np.maximum(0.0, 1 - u1))], 1)
    ax = np.argmax(np.abs(nrm), 1)
    ad = np.empty_like(local)
    for a in range(3):  # frame: normal axis a gets the cosine lobe, the other two the disc
        m = ax == a
        b, c = (a + 1) % 3, (a + 2) % 3
        ad[m, a] = local[m, 2] * nrm[m, a]
        ad[m, b] = local[m, 0]
        ad[m, c] = local[m, 1]
    ad /= np.linalg.norm(ad, axis=1, keepdims=True)
    rays = np.concatenate([pack(p, sd, 0.0, np.inf), pack(p, ad, 0.0, ao_tmax)])
    return rays, np.concatenate([src, src])
