"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

SURVEY.md §8(c) c-3 "What pins each part":
  * exact brute force on tiny volumes (tests/brute_force.py, Python Fractions);
  * closed forms: sphere column first hits (cfg1), Menger ortho hit/miss counts (cfg2),
    solid-box slab entry;
  * invariants: mirror symmetry, empty/solid volumes, non-canonical rays rejected.
A dropped term, a sign error on d<0, an off-by-one plane index or a tie broken one-sidedly
fails at least one of these.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest

import inputs
import oracle
from inputs import rays as R
import brute_force


def _occ(d):
    return inputs.dense_host(d) != 0


def _check_vs_brute(d, rays):
    occ = _occ(d)
    g = oracle.Grid.from_generator(d)
    out = g.trace(rays)
    assert (out["status"] != 2).all(), "adversarial generator produced non-canonical rays"
    bx, bt, bn = brute_force.trace(occ, rays, with_normal=True)
    np.testing.assert_array_equal(out["xyz"], bx.astype(np.int32))
    np.testing.assert_array_equal(out["normal"], bn)
    for i, te in enumerate(bt):
        if te is None:
            assert math.isinf(out["t"][i])
        else:
            # oracle t is fp32(exact); allow the double-rounding ulp
            tf = float(out["t"][i])
            assert abs(Fraction(tf) - te) <= abs(te) * Fraction(1, 2**23) + Fraction(1, 2**40), (i, tf, float(te))
    return out


@pytest.mark.parametrize("dims,p,seed", [
    ((4, 4, 4), 0.25, 1), ((5, 5, 5), 0.05, 2), ((5, 5, 5), 0.6, 3), ((7, 3, 9), 0.25, 4),
    ((8, 8, 8), 0.05, 5), ((8, 8, 8), 0.25, 6), ((8, 8, 8), 0.6, 7), ((16, 16, 16), 0.05, 8),
])
def test_oracle_equals_bruteforce_adversarial(dims, p, seed):
    d = inputs.random_occupancy(dims, p, seed)
    rays = np.concatenate([R.adversarial_rays(500, dims, seed), R.random_rays(150, dims, seed + 100)])
    out = _check_vs_brute(d, rays)
    # the adversarial set must actually exercise hits and misses
    hits = (out["status"] == 1).mean()
    assert 0.02 < hits < 0.98


def test_oracle_equals_bruteforce_axis_lattice():
    """Every axis-aligned and 45-degree lattice ray through an 8^3 random volume."""
    dims = (8, 8, 8)
    d = inputs.random_occupancy(dims, 0.15, 11)
    o, dd = [], []
    for a in range(-1, 10):
        for b in range(-1, 10):
            for dv in [(0, 0, 1), (1, 1, 1), (1, -1, 1), (0, 1, 1), (1, 0, -1), (-1, -1, -1)]:
                o.append((a, b, -2.0))
                dd.append(dv)
                o.append((a + 0.5, -2.0, b))
                dd.append((dv[2], dv[0] or 1, dv[1]))
    rays = R.pack(np.array(o, float), np.array(dd, float))
    _check_vs_brute(d, rays)


def test_sphere_closed_form_cfg1():
    """cfg1: 64^3 sphere r=28, 256^2 +z ortho rays o=((i+.5)/4,(j+.5)/4,-1).
    Column (x,y): q = 4r^2-(2x+1-R)^2-(2y+1-R)^2; hit iff q>=0 and (isqrt(q)>=1 or R odd);
    z0 = ceil((R - isqrt(q) - 1)/2); t = z0 - o_z."""
    Rr, r = 64, 28
    d = inputs.sphere(Rr, r)
    rays, perm = R.ortho(256, 256, 0.25, -1.0)
    g = oracle.Grid.from_generator(d)
    assert g.count() == 92096
    out = g.trace(rays)
    hit_cols = set()
    n_hit = 0
    for i in range(len(rays)):
        x, y = int(math.floor(rays[i, 0])), int(math.floor(rays[i, 1]))
        q = 4 * r * r - (2 * x + 1 - Rr) ** 2 - (2 * y + 1 - Rr) ** 2
        hit = q >= 0 and (math.isqrt(q) >= 1 or Rr % 2 == 1)
        if hit:
            s = math.isqrt(q)
            z0 = -((-(Rr - s - 1)) // 2)
            assert tuple(out["xyz"][i]) == (x, y, z0)
            assert out["t"][i] == np.float32(z0 + 1.0)
            hit_cols.add((x, y))
            n_hit += 1
        else:
            assert out["status"][i] == 0 and tuple(out["xyz"][i]) == (-1, -1, -1)
    assert len(hit_cols) == 2472 and n_hit == 39552


@pytest.mark.parametrize("k,R_", [(2, 9), (3, 32), (5, 256)])
def test_menger_closed_form(k, R_):
    """Level-k sponge: +z ortho rays through column centres hit 8^k columns, miss 9^k-8^k,
    and every hit is at z=0 (t = 0 - o_z)."""
    d = inputs.menger(R_, k)
    n = 3 ** k
    ys, xs = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    o = np.stack([xs.ravel() + 0.5, ys.ravel() + 0.5, np.full(n * n, -2.0)], 1)
    rays = R.pack(o, np.array([[0, 0, 1.0]]))
    g = oracle.Grid.from_generator(d)
    if k == 5:
        assert g.count() == 20 ** 5
    out = g.trace(rays)
    hits = out["status"] == 1
    assert hits.sum() == 8 ** k and (~hits).sum() == 9 ** k - 8 ** k
    assert (out["xyz"][hits, 2] == 0).all() and (out["t"][hits] == 2.0).all()


def _box_closed_form(lo, hi, dims, ray):
    """First hit on a solid box [lo,hi) inside [0,R): exact slab entry, cell tau(t+)."""
    o = [Fraction(float(ray[i])) for i in range(3)]
    dd = [Fraction(float(ray[4 + i])) for i in range(3)]
    t0 = Fraction(float(ray[3]))
    t1 = None if math.isinf(ray[7]) else Fraction(float(ray[7]))
    for a in range(3):
        if dd[a] == 0:
            if not (lo[a] <= o[a] < hi[a]):
                return None
            continue
        e = ((lo[a] if dd[a] > 0 else hi[a]) - o[a]) / dd[a]
        x = ((hi[a] if dd[a] > 0 else lo[a]) - o[a]) / dd[a]
        t0 = max(t0, e)
        t1 = x if t1 is None else min(t1, x)
    if t1 is not None and not t0 < t1:
        return None
    cell = []
    for a in range(3):
        p = o[a] + t0 * dd[a]
        if dd[a] > 0:
            c = math.floor(p)
        elif dd[a] < 0:
            c = math.ceil(p) - 1
        else:
            c = math.floor(o[a])
        cell.append(c)
    return tuple(cell), t0


def test_box_closed_form():
    dims = (24, 20, 28)
    lo, hi = (5, 3, 7), (17, 11, 20)
    d = inputs.box(dims, lo, hi)
    rays = np.concatenate([R.adversarial_rays(1500, dims, 77), R.random_rays(1500, dims, 78)])
    out = oracle.Grid.from_generator(d).trace(rays)
    for i in range(len(rays)):
        cf = _box_closed_form(lo, hi, dims, rays[i])
        if cf is None:
            assert out["status"][i] == 0, i
        else:
            assert out["status"][i] == 1 and tuple(out["xyz"][i]) == cf[0], (i, cf, out["xyz"][i])
            assert abs(Fraction(float(out["t"][i])) - cf[1]) <= abs(cf[1]) * Fraction(1, 2**23) + Fraction(1, 2**40)


def test_mirror_symmetry():
    """Mirroring volume and rays in x maps hit x -> R-1-x (catches one-sided sign handling)."""
    dims = (16, 12, 10)
    d = inputs.random_occupancy(dims, 0.1, 21)
    occ = inputs.dense_host(d)
    rays = np.concatenate([R.adversarial_rays(2000, dims, 22), R.random_rays(2000, dims, 23)])
    m = rays.copy()
    m[:, 0] = np.float32(dims[0]) - m[:, 0]
    m[:, 4] = -m[:, 4]
    m = R.canonicalize(m)
    keep = (np.float32(dims[0]) - m[:, 0]) == rays[:, 0]  # mirror exactly representable
    # half-open membership of a zero-direction axis (reading A5: cell floor(o_a)) is not
    # mirror-symmetric when o_x lies exactly on a plane; the moving-axis rule is.
    keep &= (rays[:, 4] != 0) | (rays[:, 0] != np.floor(rays[:, 0]))
    a = oracle.Grid.from_dense(occ).trace(rays[keep])
    b = oracle.Grid.from_dense(occ[:, :, ::-1]).trace(m[keep])
    hit = a["status"] == 1
    np.testing.assert_array_equal(hit, b["status"] == 1)
    np.testing.assert_array_equal(a["xyz"][hit, 0], dims[0] - 1 - b["xyz"][hit, 0])
    np.testing.assert_array_equal(a["xyz"][hit, 1:], b["xyz"][hit, 1:])
    np.testing.assert_allclose(a["t"][hit], b["t"][hit], rtol=1e-6)


def test_empty_and_solid():
    dims = (6, 5, 7)
    rays = np.concatenate([R.adversarial_rays(800, dims, 31), R.random_rays(800, dims, 32)])
    e = oracle.Grid.from_generator(inputs.empty(dims)).trace(rays)
    assert (e["status"] == 0).all() and (e["xyz"] == -1).all() and np.isinf(e["t"]).all()
    s = oracle.Grid.from_generator(inputs.solid(dims)).trace(rays)
    bx = oracle.Grid.from_generator(inputs.box(dims, (0, 0, 0), dims)).trace(rays)
    np.testing.assert_array_equal(s["xyz"], bx["xyz"])
    # solid volume: every ray that enters the box hits at its entry cell at t_start
    for i in range(len(rays)):
        cf = _box_closed_form((0, 0, 0), dims, dims, rays[i])
        assert (cf is None) == (s["status"][i] == 0)


def test_noncanonical_rejected():
    r = R.pack(np.array([[1e-30, 0.5, -1.0], [0.5, 0.5, -1.0], [0.5, 0.5, -1.0]]),
               np.array([[0, 0, 1.0], [0, 0, 1e-35], [0, 0, 3.0]]))
    r[0, 0] = np.float32(1e-30)  # bypass canonicalize
    r[1, 6] = np.float32(1e-35)
    out = oracle.Grid.from_generator(inputs.solid((4, 4, 4))).trace(r)
    assert list(out["status"]) == [2, 2, 2]


def test_procedural_equals_bitset():
    d = inputs.menger(81, 4)
    rays = R.random_rays(3000, (81, 81, 81), 5)
    a = oracle.Grid.from_generator(d).trace(rays)
    b = oracle.Grid.procedural(d).trace(rays)
    np.testing.assert_array_equal(a["xyz"], b["xyz"])
    np.testing.assert_array_equal(a["t"], b["t"])


def test_sparse_rasteriser_matches_generator():
    """G5 bitset (per-object rasteriser) vs the brute-force lowest-k definition on a sample."""
    d = inputs.sparse(384, 0x4096)
    g = oracle.Grid.from_generator(d)
    dense = inputs.dense_host(d) != 0          # binned evaluator (inputs/volgen_lib.cu)
    assert g.count() == int(dense.sum()) > 1000
    zs, ys, xs = np.nonzero(dense)
    rng = np.random.default_rng(0)
    idx = rng.choice(len(xs), 300, replace=False)
    for x, y, z in zip(xs[idx], ys[idx], zs[idx]):
        assert g.get(x, y, z) == 1
        assert inputs.voxel_host(d, x, y, z) != 0   # brute-force lowest-k definition
    for x, y, z in rng.integers(0, 384, size=(300, 3)):
        assert g.get(x, y, z) == (inputs.voxel_host(d, x, y, z) != 0) == bool(dense[z, y, x])


def test_procedural_sparse_equals_bitset():
    d = inputs.sparse(384, 0x4096)
    rays = np.concatenate([R.random_rays(6000, (384,) * 3, 3), R.adversarial_rays(2000, (384,) * 3, 4)])
    a = oracle.Grid.from_generator(d).trace(rays)
    b = oracle.Grid.procedural(d).trace(rays)
    assert (a["status"] == 1).sum() > 50
    np.testing.assert_array_equal(a["xyz"], b["xyz"])
    np.testing.assert_array_equal(a["t"], b["t"])


def _negative_tmin_rays(dims, seed, n=600):
    """Rays whose segment starts behind the origin (tmin < 0; reading R5): origins inside and
    outside the box, tmin in [-2R, 0), finite and infinite tmax (some tmax < 0 too)."""
    rng = np.random.Generator(np.random.MT19937(seed))
    R_ = np.asarray(dims, dtype=np.float64)
    o = np.round((rng.random((n, 3)) * 1.4 - 0.2) * R_ * 16) / 16
    d = rng.integers(-3, 4, size=(n, 3)).astype(np.float64)
    d[np.abs(d).sum(1) == 0] = (1, 1, 1)
    g = rng.normal(size=(len(d[::3]), 3))
    d[::3] = 2 * g / np.linalg.norm(g, axis=1, keepdims=True)  # |d_a| <= 1 after the halving below
    tmin = -np.round(rng.random(n) * 2 * R_.max() * 8) / 8 - 0.125
    tmax = np.where(rng.random(n) < 0.5, np.inf, tmin + np.round(rng.random(n) * R_.max() * 8) / 8 + 0.125)
    return R.pack(o, d / 2, tmin, tmax)


@pytest.mark.parametrize("dims,p,seed", [((8, 8, 8), 0.1, 41), ((6, 9, 5), 0.3, 42)])
def test_negative_tmin_vs_bruteforce(dims, p, seed):
    """tmin < 0 (the GPU hung on such rays): the oracle walks [tmin, tmax) behind the
    origin exactly as the brute-force slab test defines it."""
    d = inputs.random_occupancy(dims, p, seed)
    rays = _negative_tmin_rays(dims, seed)
    assert (rays[:, 3] < 0).all()
    out = _check_vs_brute(d, rays)
    assert 0.05 < (out["status"] == 1).mean() < 0.95


# ---- exact brute force at scale: >= 1e5 rays per size, 4^3 .. 32^3 (tests/brute/brute.c) -----
def _brute_rays(dims, seed, n):
    import test_oracle as T
    k = n // 3
    return np.concatenate([R.adversarial_rays(k, dims, seed), R.random_rays(k, dims, seed + 1),
                           T._negative_tmin_rays(dims, seed + 2, n - 2 * k)])


def _assert_oracle_equals_brute(d, rays, label):
    import brute
    occ = inputs.dense_host(d) != 0
    out = oracle.Grid.from_generator(d).trace(rays)
    b = brute.trace(occ, rays)
    assert (b["status"] != 3).all(), f"{label}: non-unique minimum entry time (contradicts reading A21)"
    assert (b["status"] != 2).all() and (out["status"] != 2).all(), label
    np.testing.assert_array_equal(out["status"], b["status"], err_msg=label)
    np.testing.assert_array_equal(out["xyz"], b["xyz"], err_msg=label)
    hit = b["status"] == 1
    # exact t = tnum / tden * 2^14; the oracle's fp32 t must be its correctly rounded value
    # (within half an fp32 ulp, plus the float64 evaluation of the exact fraction)
    te = np.ldexp(b["tnum"][hit].astype(np.float64) / b["tden"][hit].astype(np.float64), 14)
    tf = out["t"][hit].astype(np.float64)
    assert np.all(np.abs(tf - te) <= np.abs(te) * 2.0 ** -24 * (1 + 2.0 ** -20) + 2.0 ** -60), label
    assert np.isinf(out["t"][~hit]).all()
    # entry face: lowest entry axis, -sign(d_a)
    nrm = np.zeros((len(rays), 3), np.int8)
    for a in (2, 1, 0):
        m = hit & ((b["axes"] >> a) & 1).astype(bool)
        nrm[m] = 0
        nrm[m, a] = np.where(rays[m, 4 + a] > 0, -1, 1)
    np.testing.assert_array_equal(out["normal"], nrm, err_msg=label)
    return hit.mean()


@pytest.mark.parametrize("R_", [4, 8, 16, 32])
def test_oracle_equals_bruteforce_1e5_rays(R_):
    """SURVEY §8(c) c-3 row 'Semantics': exact brute force on R^3 random volumes (p in 0.05 / 0.25 /
    0.6), 102,000 rays per size (adversarial lattice, random inside/outside, tmin < 0), 100 %."""
    dims = (R_, R_, R_)
    for j, p in enumerate((0.05, 0.25, 0.6)):
        d = inputs.random_occupancy(dims, p, 900 + 10 * R_ + j)
        rate = _assert_oracle_equals_brute(d, _brute_rays(dims, 7 * R_ + j, 34000), f"{R_}^3 p={p}")
        assert 0.02 < rate < 0.99


# ---- occupancy helpers of the oracle, pinned per voxel ------------------
def _aabb_faces(objs, R_):
    """Every voxel of the outermost layer (6 faces) of every G5 object's AABB [c-r, c+r)^3,
    clipped to [0, R)^3: exactly the voxels a bin range one short at either end would drop."""
    pts = []
    for cx, cy, cz, r, _, _ in objs:
        c = np.array([cx, cy, cz], np.int64)
        lo, hi = np.maximum(c - r, 0), np.minimum(c + r, R_)  # [lo, hi)
        if np.any(hi <= lo):
            continue
        for a in range(3):
            for plane in (c[a] - r, c[a] + r - 1):
                if not (0 <= plane < R_):
                    continue
                b, e = [x for x in range(3) if x != a]
                u, v = np.meshgrid(np.arange(lo[b], hi[b]), np.arange(lo[e], hi[e]), indexing="ij")
                p = np.empty((u.size, 3), np.int64)
                p[:, a], p[:, b], p[:, e] = plane, u.ravel(), v.ravel()
                pts.append(p)
    return np.concatenate(pts)


def test_sparse_occupancy_aabb_faces_4096():
    """G5 at full size (cfg5): the procedural (64^3-binned) occupancy, the per-object rasterised
    bitset and the input library's own binned evaluator agree on every voxel of every object's
    AABB boundary — the voxels an off-by-one bin range (lo = c-r+1, hi = c+r-2) would lose."""
    d = inputs.sparse(4096, 0x4096)
    objs = inputs.sparse_objects(0x4096)
    pts = _aabb_faces(objs, 4096)
    a = oracle.Grid.procedural(d).get_many(pts)
    g = oracle.Grid.from_generator(d)
    b = g.get_many(pts)
    g.close()
    c = (inputs.voxels_host(d, pts) != 0).astype(np.uint8)
    assert len(pts) > 10_000_000 and 0.05 < c.mean() < 0.9
    np.testing.assert_array_equal(a, c)
    np.testing.assert_array_equal(b, c)
    # a sample against the brute-force lowest-k definition (every object tested)
    rng = np.random.default_rng(5)
    for i in rng.choice(len(pts), 200, replace=False):
        assert (inputs.voxel_host(d, *pts[i]) != 0) == bool(c[i])


@pytest.mark.parametrize("R_,lo,ext", [(512, (0, 0, 0), (512, 512, 512)), (4096, (1920, 1920, 1920), (256, 256, 256)),
                                       (4096, (3840, 0, 3840), (256, 256, 256))])
def test_sparse_occupancy_whole_box(R_, lo, ext):
    """Per-voxel equality over whole boxes: procedural vs rasterised vs the input evaluator."""
    d = inputs.sparse(R_, 0x4096)
    a = oracle.Grid.procedural(d).box(lo, ext)
    g = oracle.Grid.from_generator(d)
    b = g.box(lo, ext)
    g.close()
    z, y, x = np.meshgrid(*[np.arange(lo[k], lo[k] + ext[k]) for k in (2, 1, 0)], indexing="ij")
    c = (inputs.voxels_host(d, np.stack([x.ravel(), y.ravel(), z.ravel()], 1)) != 0).astype(np.uint8)
    c = c.reshape(a.shape)
    assert c.sum() > 1000
    np.testing.assert_array_equal(a, c)
    np.testing.assert_array_equal(b, c)


@pytest.mark.parametrize("mk", [lambda: inputs.solid((13, 7, 5)), lambda: inputs.box((13, 7, 5), (9, 3, 1), (13, 7, 5)),
                                lambda: inputs.random_occupancy((13, 7, 5), 0.5, 3),
                                lambda: inputs.random_occupancy((64, 64, 64), 0.3, 4)])
def test_from_dense_equals_generator_every_voxel(mk):
    """oracle_grid_from_dense (dense RGBA input) == the generator's bitset on every voxel,
    including the last one (x,y,z) = (Rx-1, Ry-1, Rz-1)."""
    d = mk()
    dense = inputs.dense_host(d)
    a = oracle.Grid.from_dense(dense).box((0, 0, 0), inputs.dims_of(d))
    b = oracle.Grid.from_generator(d).box((0, 0, 0), inputs.dims_of(d))
    np.testing.assert_array_equal(a, (dense != 0).astype(np.uint8))
    np.testing.assert_array_equal(b, (dense != 0).astype(np.uint8))


def test_slab_counts_equal_dense_slab_sums():
    """oracle_grid_slab_counts (c-2 step 1's cross-check) == per-z-slab sums of the input array."""
    for d in (inputs.random_occupancy((24, 20, 28), 0.3, 8), inputs.sphere(64, 28), inputs.menger(81, 4)):
        dense = inputs.dense_host(d) != 0
        for g in (oracle.Grid.from_generator(d), oracle.Grid.procedural(d), oracle.Grid.from_dense(inputs.dense_host(d))):
            sc = g.slab_counts()
            np.testing.assert_array_equal(sc, dense.sum(axis=(1, 2)))
        assert oracle.Grid.from_generator(d).count() == int(dense.sum())
