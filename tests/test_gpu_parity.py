"""GPU parity: the CUDA path through the C ABI (libvf.so) vs the CPU oracle, element by element.

Every hybrid format must return the oracle's first-hit voxel bit for bit and the miss flag
exactly, t within 1e-4 relative (north_star). Volumes and rays are the
seeded synthetic inputs of inputs/ (SURVEY.md §8(d)); the oracle never sees GPU output.
"""
from __future__ import annotations

import numpy as np
import pytest

import inputs
import oracle
from inputs import rays as R
from parity import assert_parity, gpu_trace

pytestmark = pytest.mark.gpu


def _vf():
    from paper_2410_14128_b200 import vf
    return vf


def _dense_dev(d):
    import torch
    return torch.from_numpy(inputs.dense_host(d).view(np.int32)).cuda()


def _rays_small(dims, seed, n_adv=3000, n_rand=2000):
    return np.concatenate([R.adversarial_rays(n_adv, dims, seed), R.random_rays(n_rand, dims, seed + 1)])


# ---------------------------------------------------------------- cfg1: Raw single level
def test_cfg1_sphere_raw():
    vf = _vf()
    d = inputs.sphere(64, 28)
    h = vf.build(_dense_dev(d), "R(6, 6, 6)")
    g = oracle.Grid.from_generator(d)
    ortho, _ = R.ortho(256, 256, 0.25, -1.0)
    obl, _ = R.ortho(256, 256, 0.25, -1.0, direction=(0.25, 0.5, 1.0))
    for name, rays in [("ortho", ortho), ("oblique", obl), ("adversarial", _rays_small((64,) * 3, 5))]:
        ref = g.trace(rays)
        for restart in (False, True):
            xyz, t = gpu_trace(h, rays, restart)
            assert_parity(xyz, t, ref, f"cfg1 {name} restart={restart}")
    s = h.stats()
    assert s["nonempty_voxels"] == 92096 and s["bytes_used"] == 4 * (4 + 64 ** 3)


# ---------------------------------------------------------------- many formats, small volumes
SMALL_FORMATS_16 = [
    "R(4, 4, 4)", "S(4)", "G(4)", "T(2, 2)", "T(1, 4)", "R(2^3) G(2)", "R(1^3) S(3)", "G(2) R(2^3)",
    "S(2) R(2, 2, 2)", "T(2, 1) R(2^3)", "T(2, 1) T(1, 1) R(1^3)", "R(1, 1, 1) T(2, 1) S(1)",
    "R(1^3) S(1) G(1) T(1, 1)", "G(1) T(2, 1) R(1^3)", "R(2^3) R(2^3)", "S(1) S(1) S(1) S(1)",
    "G(3) G(1)", "T(2, 1) T(2, 1)",
    "D(4, 4, 4, 3)", "D(2^3, 2) G(2)", "R(1^3) D(3^3, 6)", "D(2^3, 6) D(2^3, 1)", "S(2) D(2^3, 4)",
]


@pytest.mark.parametrize("fmt", SMALL_FORMATS_16)
@pytest.mark.parametrize("p", [0.03, 0.3])
def test_small_formats_vs_oracle(fmt, p):
    vf = _vf()
    dims = (16, 16, 16)
    d = inputs.random_occupancy(dims, p, 1234 + int(p * 100))
    h = vf.build(_dense_dev(d), fmt)
    rays = _rays_small(dims, 99)
    ref = oracle.Grid.from_generator(d).trace(rays)
    for restart in (False, True):
        for pers in (False, True):
            xyz, t = gpu_trace(h, rays, restart, pers)
            assert_parity(xyz, t, ref, f"{fmt} p={p} restart={restart} persistent={pers}")


@pytest.mark.parametrize("fmt,dims", [
    ("R(2, 1, 3) G(2)", (16, 8, 32)), ("R(0, 2, 1) S(3)", (8, 32, 16)), ("R(3, 0, 1) T(2, 1) R(1^3)", (64, 8, 16)),
    ("R(1, 2, 0) R(2^3)", (8, 16, 4)), ("D(1, 2, 0, 3) R(2^3)", (8, 16, 4)), ("D(3, 1, 2, 6) G(2)", (32, 8, 16)),
])
def test_noncubic_first_level(fmt, dims):
    vf = _vf()
    d = inputs.random_occupancy(dims, 0.1, 77)
    h = vf.build(_dense_dev(d), fmt)
    rays = _rays_small(dims, 7)
    ref = oracle.Grid.from_generator(d).trace(rays)
    for restart in (False, True):
        xyz, t = gpu_trace(h, rays, restart)
        assert_parity(xyz, t, ref, f"{fmt} restart={restart}")


# ---------------------------------------------------------------- cfg2: 256^3 Menger
CFG2_FORMATS = ["S(8)", "G(8)", "G(5) R(3, 3, 3)", "T(2, 4)", "R(8, 8, 8)", "R(3^3) G(5)", "D(4^3, 6) G(4)",
                "D(8^3, 6)", "D(3^3, 6) D(3^3, 6) R(2^3)"]


@pytest.mark.parametrize("fmt", CFG2_FORMATS)
def test_cfg2_menger(fmt):
    import torch
    vf = _vf()
    d = inputs.menger(256, 5)
    keys, rgba = inputs.voxels_device(d)
    h = vf.build((keys, rgba, (256, 256, 256)), fmt)
    g = oracle.Grid.from_generator(d)
    persp, _ = R.camera("menger", scale=4)        # 256 x 256 subsample of the 1024^2 camera
    tunnel, _ = R.camera("menger_tunnel", scale=8)
    n = 3 ** 5
    ys, xs = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ax = R.pack(np.stack([xs.ravel() + 0.5, ys.ravel() + 0.5, np.full(n * n, -2.0)], 1), np.array([[0, 0, 1.0]]))
    for name, rays in [("persp", persp), ("tunnel", tunnel), ("axis", ax), ("adv", _rays_small((256,) * 3, 3, 2000, 1000))]:
        ref = g.trace(rays)
        for restart in (False, True):
            xyz, t = gpu_trace(h, rays, restart)
            assert_parity(xyz, t, ref, f"cfg2 {fmt} {name} restart={restart}")
    assert h.stats()["nonempty_voxels"] == 20 ** 5
    del torch


# ---------------------------------------------------------------- build: query / sizes
@pytest.mark.parametrize("fmt", ["R(4, 4, 4)", "S(4)", "G(4)", "T(2, 2)", "R(2^3) G(2)", "G(1) T(2, 1) R(1^3)",
                                 "R(1^3) S(1) G(1) T(1, 1)"])
def test_query_equals_dense(fmt):
    import torch
    vf = _vf()
    dims = (16, 16, 16)
    d = inputs.random_occupancy(dims, 0.2, 5)
    dense = inputs.dense_host(d)
    h = vf.build(torch.from_numpy(dense.view(np.int32)).cuda(), fmt)
    zz, yy, xx = np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij")
    xyz = torch.from_numpy(np.stack([xx.ravel(), yy.ravel(), zz.ravel()], 1).astype(np.int32)).cuda()
    got = h.query(xyz).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got, dense.ravel())


def test_size_closed_forms():
    """SURVEY.md §8(c) c-3 'Bytes' row (paper layout, word 0 included)."""
    import torch
    vf = _vf()

    def words(fmt, d, flags=vf.VF_BUILD_DEFAULT):
        h = vf.build(torch.from_numpy(inputs.dense_host(d).view(np.int32)).cuda(), fmt, flags)
        return h.stats()["paper_layout_bytes"] // 4

    L = 4
    R_ = 2 ** L
    solid = inputs.solid((R_,) * 3)
    one = inputs.single((R_,) * 3, (3, 9, 14))
    empty = inputs.empty((R_,) * 3)
    assert words(f"S({L})", empty) == 1 and words(f"G({L})", empty) == 1   # buffer [0]
    assert words(f"S({L})", solid) == 1 + 2 * (8 ** (L + 1) - 1) // 7
    assert words(f"G({L})", solid) == 1 + 9 * L + 1                          # L internal + 1 leaf
    assert words(f"S({L})", one) == 1 + 2 * (L + 1)
    assert words(f"G({L})", one) == 1 + 2 * L + 1
    assert words("T(2, 2)", solid) == 1 + 4 * (64 ** 2 - 1) // 63 + 64 ** 2
    assert words("T(2, 2)", one) == 1 + 4 * 2 + 1
    assert words(f"R({L}, {L}, {L})", one) == 1 + R_ ** 3
    # whole-level dedup never adds storage
    rnd = inputs.random_occupancy((R_,) * 3, 0.3, 9)
    for fmt in ["R(2^3) G(2)", "R(1^3) G(3)", "G(2) G(2)"]:
        assert words(fmt, rnd, vf.VF_BUILD_WHOLE_LEVEL_DEDUP) <= words(fmt, rnd, 0)


def test_empty_volume_all_miss():
    import torch
    vf = _vf()
    dims = (8, 8, 8)
    for fmt in ["R(3, 3, 3)", "G(3)", "S(3)", "T(1, 3)", "R(1^3) G(2)"]:
        h = vf.build(torch.zeros((8, 8, 8), dtype=torch.int32, device="cuda"), fmt)
        assert h.stats()["root"] == 0 and h.bytes_used == 4
        rays = _rays_small(dims, 1, 300, 300)
        xyz, t = gpu_trace(h, rays)
        assert (xyz == -1).all() and np.isinf(t).all()


def test_format_errors():
    import torch
    vf = _vf()
    v = torch.zeros((16, 16, 16), dtype=torch.int32, device="cuda")
    with pytest.raises(vf.VfError) as e:
        vf.build(v, "R(2, 2, 2) R(1, 2, 1)")
    assert e.value.status == vf.VF_ERR_FORMAT
    with pytest.raises(vf.VfError) as e:
        vf.build(v, "R(1, 1, 1) D(1, 2, 1, 6) G(1)")
    assert e.value.status == vf.VF_ERR_FORMAT
    with pytest.raises(vf.VfError) as e:
        vf.build(v, "G(5)")
    assert e.value.status == vf.VF_ERR_FORMAT


def test_counters_consistent():
    """The counting variant returns the same hits and sane per-ray work counts."""
    import torch
    vf = _vf()
    d = inputs.menger(256, 5)
    keys, rgba = inputs.voxels_device(d)
    rays, _ = R.camera("menger", scale=4)
    rt = torch.from_numpy(rays).cuda()
    for fmt, fields in [("G(5) R(3, 3, 3)", ("svdag_nodes", "raw_cells")), ("S(8)", ("svo_nodes",)),
                        ("T(2, 4)", ("ntree_nodes",))]:
        h = vf.build((keys, rgba, (256, 256, 256)), fmt)
        a = h.trace(rt).cpu().numpy()
        hits = torch.empty_like(rt[:, :4].contiguous().view(torch.int32))
        c = h.counters(rt, hits)
        np.testing.assert_array_equal(hits.cpu().numpy(), a)
        n = len(rays)
        assert c["rays"] == n and c["hits"] == int((a[:, 0] >= 0).sum())
        for f in fields:
            assert c[f] > 0
        per = 4 * (c["raw_cells"] + c["svdag_nodes"] + c["svdag_ptrs"] + c["leaf_words"]) + 8 * c["svo_nodes"] + \
            16 * c["ntree_nodes"]
        assert c["format_bytes"] == per
        assert c["exact_calls"] < 0.05 * n


def test_trace_host_matches_device():
    import torch
    vf = _vf()
    d = inputs.random_occupancy((32, 32, 32), 0.05, 3)
    h = vf.build(_dense_dev(d), "R(2^3) G(3)")
    rays = R.random_rays(5000, (32, 32, 32), 4)
    xyz, t = gpu_trace(h, rays)
    hr = torch.from_numpy(rays).pin_memory()
    hh = torch.empty((len(rays), 4), dtype=torch.int32).pin_memory()
    h.trace_host(hr, hh)
    out = hh.numpy()
    np.testing.assert_array_equal(out[:, :3], xyz)
    np.testing.assert_array_equal(out[:, 3].view(np.float32), t)


# ---------------------------------------------------------------- DF distance field
@pytest.mark.parametrize("fmt,M", [("D(4, 4, 4, 5)", 5), ("R(1^3) D(3^3, 6)", 6), ("D(4, 3, 4, 2)", 2)])
def test_df_distances_are_exact_l1(fmt, M):
    """Every DF cell stores min(M, L1 distance to the nearest non-empty cell of its grid)
    (PAPER.md:59, :100-105): checked against a brute-force L1 distance transform."""
    import torch
    vf = _vf()
    L = vf.parse_format(fmt)
    dims = vf.format_resolution(L)
    d = inputs.random_occupancy(dims, 0.02, 31)
    dense = inputs.dense_host(d)
    h = vf.build(torch.from_numpy(dense.view(np.int32)).cuda(), fmt)
    words = h.buffer_words()
    Rx, Ry, Rz = dims
    # locate the DF grids: single level -> one grid at word[0]; R(1^3) D(..) -> 8 sub-grid pointers
    if fmt.startswith("D"):
        grids = [(words[0], (0, 0, 0), (Rx, Ry, Rz))]
    else:
        top = words[0]
        e = Rx // 2
        grids = []
        for z in range(2):
            for y in range(2):
                for x in range(2):
                    ptr = words[top + x + 2 * (y + 2 * z)]
                    if ptr:
                        grids.append((ptr, (x * e, y * e, z * e), (e, e, e)))
    assert grids
    for ptr, o, ext in grids:
        sub = dense[o[2]:o[2] + ext[2], o[1]:o[1] + ext[1], o[0]:o[0] + ext[0]] != 0
        occ = np.argwhere(sub)  # (z, y, x)
        zz, yy, xx = np.meshgrid(np.arange(ext[2]), np.arange(ext[1]), np.arange(ext[0]), indexing="ij")
        cells = np.stack([zz.ravel(), yy.ravel(), xx.ravel()], 1)
        dist = np.abs(cells[:, None, :] - occ[None, :, :]).sum(-1).min(1)
        expect = np.minimum(dist, M)
        n = ext[0] * ext[1] * ext[2]
        got = words[ptr:ptr + 2 * n].reshape(n, 2)
        np.testing.assert_array_equal(got[:, 1], expect, err_msg=fmt)
        np.testing.assert_array_equal(got[:, 0], dense[o[2]:o[2] + ext[2], o[1]:o[1] + ext[1],
                                                        o[0]:o[0] + ext[0]].ravel())


# ---------------------------------------------------------------- the paper's Table 2 (all 40 formats)
def _table2():
    import os
    rows = []
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "table2_formats.txt")):
        if line.startswith("#") or not line.strip():
            continue
        label, res, sig = line.strip().split(" ", 2)
        rows.append((int(label), int(res), sig))
    return rows


@pytest.mark.parametrize("res", [512, 2048])
def test_table2_formats_parity(res):
    """Every format of PAPER.md Table 2 (rows 1-20 at 2048^3 on the cfg4 city, rows 21-40 at
    512^3 on the t512 city), stack and restart, against the oracle on every ray of the frame."""
    import torch
    import bench
    vf = _vf()
    cfg = "cfg4" if res == 2048 else "t512"
    vol = bench.make_volume(bench.CONFIGS[cfg][0])
    keys, rgba = inputs.voxels_device(vol)
    rays, _ = bench.make_rays(cfg)
    idx = np.arange(len(rays))  # every ray of the frame
    ref = oracle.Grid.from_generator(vol).trace(rays)
    rt = torch.from_numpy(rays).cuda()
    for label, r, sig in _table2():
        if r != res:
            continue
        h = vf.build((keys, rgba, inputs.dims_of(vol)), sig)
        for restart in (False, True):
            out = h.trace(rt, restart=restart).cpu().numpy()
            assert_parity(out[idx, :3], out[idx, 3].view(np.float32), ref, f"Table 2 row {label} {sig} restart={restart}")
        h.close()


# ---------------------------------------------------------------- closest-hit payload (NEXT 4)
@pytest.mark.parametrize("fmt", ["R(4, 4, 4)", "G(4)", "S(2) R(2^3)", "T(2, 2)", "R(1^3) D(3^3, 3)", "G(2) T(1, 2)"])
def test_payload_rgba_and_entry_face(fmt):
    """rgba = the stored voxel at the hit (the dense grid); normal = the oracle's entry face
    (pinned to the brute force's geometric definition)."""
    import torch
    vf = _vf()
    dims = (16, 16, 16)
    d = inputs.random_occupancy(dims, 0.1, 8)
    dense = inputs.dense_host(d)
    h = vf.build(torch.from_numpy(dense.view(np.int32)).cuda(), fmt)
    rays = _rays_small(dims, 17)
    ref = oracle.Grid.from_generator(d).trace(rays)
    rt = torch.from_numpy(rays).cuda()
    for restart in (False, True):
        hits, pay = h.trace_payload(rt, restart=restart)
        hits, pay = hits.cpu().numpy(), pay.cpu().numpy()
        assert_parity(hits[:, :3], hits[:, 3].view(np.float32), ref, fmt)
        hit = ref["xyz"][:, 0] >= 0
        x, y, z = ref["xyz"][hit].T
        np.testing.assert_array_equal(np.ascontiguousarray(pay[hit, 0]).view(np.uint32), dense[z, y, x])
        assert (pay[~hit] == 0).all()
        nrm = np.ascontiguousarray(pay[:, 1]).view(np.uint8).reshape(-1, 4)[:, :3].view(np.int8)
        np.testing.assert_array_equal(nrm, ref["normal"])


# ---------------------------------------------------------------- compiled-in formats (Lane SPEC)
@pytest.mark.parametrize("fmt,dims", [("R(2^3) G(3)", 32), ("R(1^3) G(4)", 32), ("G(2) R(2^3)", 16),
                                      ("T(1, 1) T(1, 2) R(1^3)", 16), ("G(4)", 16), ("T(1, 4)", 16),
                                      ("R(2^3) T(1, 3)", 32), ("S(2) G(2)", 16), ("R(1^3) G(1) S(2)", 16),
                                      ("D(2^3, 3) G(2)", 16), ("R(4^3)", 16), ("D(4^3, 3)", 16)])
@pytest.mark.parametrize("p", [0.02, 0.3])
def test_compiled_in_format_vs_oracle(fmt, dims, p):
    """Formats with a compiled-in kernel (trace.cu select_spec: R(A^3) G(M) as arithmetic in the
    tier index, other listed formats as packed compile-time tier tables). Same oracle parity as the
    generic kernel, stack and restart, payload included; the generic kernel (VF_NO_SPEC,
    subprocess) returns the same bits."""
    import os
    import subprocess
    import sys
    import torch
    vf = _vf()
    d = inputs.random_occupancy((dims,) * 3, p, 4321)
    dense = inputs.dense_host(d)
    h = vf.build(torch.from_numpy(dense.view(np.int32)).cuda(), fmt)
    rays = np.concatenate([R.adversarial_rays(6000, (dims,) * 3, 3), R.random_rays(4000, (dims,) * 3, 4)])
    ref = oracle.Grid.from_generator(d).trace(rays)
    rt = torch.from_numpy(rays).cuda()
    outs = []
    for restart in (False, True):
        hits, pay = h.trace_payload(rt, restart=restart)
        hits, pay = hits.cpu().numpy(), pay.cpu().numpy()
        assert_parity(hits[:, :3], hits[:, 3].view(np.float32), ref, f"{fmt} restart={restart}")
        hit = ref["xyz"][:, 0] >= 0
        x, y, z = ref["xyz"][hit].T
        np.testing.assert_array_equal(np.ascontiguousarray(pay[hit, 0]).view(np.uint32), dense[z, y, x])
        out = h.trace(rt, restart=restart).cpu().numpy()
        np.testing.assert_array_equal(out, hits)
        outs.append(out)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np, torch; sys.path.insert(0, sys.argv[1]); import inputs; "
            "from paper_2410_14128_b200 import vf; d = inputs.random_occupancy((%d,) * 3, %r, 4321); "
            "h = vf.build(torch.from_numpy(inputs.dense_host(d).view(np.int32)).cuda(), %r); "
            "r = torch.from_numpy(np.load(sys.argv[2])).cuda(); "
            "np.save(sys.argv[3], np.stack([h.trace(r, restart=s).cpu().numpy() for s in (False, True)]))"
            % (dims, p, fmt))
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        np.save(os.path.join(td, "r.npy"), rays)
        rr = subprocess.run([sys.executable, "-c", code, root, os.path.join(td, "r.npy"), os.path.join(td, "o.npy")],
                            env=dict(os.environ, VF_NO_SPEC="1"), capture_output=True, text=True, timeout=300)
        assert rr.returncode == 0, rr.stderr[-2000:]
        gen = np.load(os.path.join(td, "o.npy"))
    np.testing.assert_array_equal(gen[0], outs[0])
    np.testing.assert_array_equal(gen[1], outs[1])


# ---------------------------------------------------------------- rays behind the origin, bad rays
@pytest.mark.parametrize("fmt", ["R(4, 4, 4)", "R(2^3) G(2)", "S(4)", "T(2, 2)", "D(2^3, 2) G(2)", "G(1) T(2, 1) R(1^3)"])
def test_negative_tmin_parity_and_termination(fmt):
    """with tmin < 0 the step's certification threshold m(1 + eps) fell below m
    and the walk never advanced. Every such ray must now terminate with the oracle's answer."""
    import test_oracle
    vf = _vf()
    dims = (16, 16, 16)
    d = inputs.random_occupancy(dims, 0.08, 5)
    h = vf.build(_dense_dev(d), fmt)
    rays = np.concatenate([test_oracle._negative_tmin_rays(dims, 3, 4000),
                           R.pack(np.array([[5.5, 3.25, 7.75]]), np.array([[1.0, 0, 0]]), -1.0, np.inf)])
    ref = oracle.Grid.from_generator(d).trace(rays)
    assert (ref["status"] != 2).all()
    for restart in (False, True):
        xyz, t = gpu_trace(h, rays, restart)
        assert_parity(xyz, t, ref, f"{fmt} tmin<0 restart={restart}")


def test_nonfinite_rays_miss():
    """Non-finite origin / direction / tmin or NaN tmax: a miss (vf.h), never a hang."""
    vf = _vf()
    d = inputs.solid((8, 8, 8))
    h = vf.build(_dense_dev(d), "R(1^3) G(2)")
    nan, inf = np.float32(np.nan), np.float32(np.inf)
    base = np.array([1.5, 1.5, -1.0, 0.0, 0.0, 0.0, 1.0, inf], dtype=np.float32)
    rays = np.tile(base, (8, 1))
    rays[0, 0] = nan
    rays[1, 4] = inf
    rays[2, 3] = -inf
    rays[3, 3] = nan
    rays[4, 7] = nan
    rays[5, 1] = inf
    rays[6, 6] = nan
    xyz, t = gpu_trace(h, rays)
    assert (xyz[:7] == -1).all() and np.isinf(t[:7]).all()
    assert tuple(xyz[7]) == (1, 1, 0)  # the unmodified ray hits


# ---------------------------------------------------------------- VF_BUILD_ALIGN_NODES (a6 option ii)
@pytest.mark.parametrize("fmt,R_", [("R(2^3) G(3)", 32), ("R(4^3) G(7)", 2048)])
def test_align_nodes_parity_and_bytes(fmt, R_):
    """SVDAG nodes padded to 16-B multiples: the
    same first hits as the oracle (stack and restart, through the aligned-header kernel), the same
    paper-layout bytes as the packed build, more device bytes, and every internal node 16-B
    aligned (its child pointers, read back from the buffer, are multiples of 4 words)."""
    import torch
    vf = _vf()
    if R_ == 32:
        d = inputs.random_occupancy((32,) * 3, 0.05, 0xA11)
        rays = _rays_small((32,) * 3, 61)
    else:
        d = inputs.city(2048)
        rays = R.camera("city", scale=4)[0]
    keys, rgba = inputs.voxels_device(d)
    hp = vf.build((keys, rgba, inputs.dims_of(d)), fmt)
    ha = vf.build((keys, rgba, inputs.dims_of(d)), fmt, flags=vf.VF_BUILD_DEFAULT | vf.VF_BUILD_ALIGN_NODES)
    sp, sa = hp.stats(), ha.stats()
    assert sa["paper_layout_bytes"] == sp["paper_layout_bytes"] and sa["bytes_used"] > sp["bytes_used"]
    assert sa["compiled_in"]
    # the top Raw grid's non-zero cells are SVDAG root pointers: all 16-B aligned
    top = ha.buffer_words(sa["root"], 8 ** int(fmt[2]) if R_ == 32 else 16 ** 3)
    assert top.any() and (top[top != 0] % 4 == 0).all()
    g = oracle.Grid.from_generator(d)
    ref = g.trace(rays)
    for restart in (False, True):
        xyz, t = gpu_trace(ha, rays, restart)
        assert_parity(xyz, t, ref, f"{fmt} aligned restart={restart}")
        xp, tp = gpu_trace(hp, rays, restart)
        assert np.array_equal(xyz, xp) and np.array_equal(t.view(np.int32), tp.view(np.int32))
    hp.close()
    ha.close()
    del keys, rgba
    torch.cuda.empty_cache()


def test_trace_scatter_equals_trace_unpermuted():
    """vf_trace_scatter (the fused trace + gather's kernel path) stores the hit of ray i at
    slots[i]: on a local buffer with slots = the rays' pixel indices it must produce exactly
    vf_trace's hits, un-permuted into pixel order (stack and restart; the ragged last tile
    included: 72x40 pixels)."""
    import torch
    vf = _vf()
    d = inputs.menger(128, 4)
    keys, rgba = inputs.voxels_device(d)
    h = vf.build((keys, rgba, (128,) * 3), "R(3^3) G(4)")
    rays, perm = R.perspective(72, 40, 60.0, (-40.3, 60.7, -70.1), (40.5, 40.5, 40.5))
    rt = torch.from_numpy(rays).cuda()
    slots = torch.from_numpy(perm.astype(np.int32)).cuda()
    for restart in (False, True):
        ref = h.trace(rt, restart=restart).cpu().numpy()
        frame = torch.full((len(rays), 4), 0x7F7F7F7F, dtype=torch.int32, device="cuda")
        h.trace_scatter(rt, frame, slots, restart=restart)
        out = frame.cpu().numpy()
        assert np.array_equal(out[perm], ref)
    h.close()


_COUNT_CHILD = r'''
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import inputs
from inputs import rays as R
from paper_2410_14128_b200 import vf
kind, fmt = sys.argv[1], sys.argv[2]
d = inputs.random_occupancy((32,) * 3, 0.05, 0xC0) if kind == "rand" else inputs.menger(256, 5)
dims = inputs.dims_of(d)
keys, rgba = inputs.voxels_device(d)
h = vf.build((keys, rgba, dims), fmt)
rays = np.concatenate([R.adversarial_rays(3000, dims, 71), R.random_rays(3000, dims, 72)])
rt = torch.from_numpy(rays).cuda()
print(json.dumps([h.counters(rt, restart=r) for r in (False, True)]))
'''


@pytest.mark.parametrize("kind,fmt", [("rand", "R(2^3) G(3)"), ("menger", "G(5) R(3^3)")])
def test_counting_runs_the_compiled_in_traversal(kind, fmt):
    """vf_trace_counters of a headline format runs the compiled-in kernel (the code bench.py times),
    and every per-ray counter (cells, steps, descents, format bytes, sector reads, distinct words,
    exact fallbacks) equals the generic tier-table kernel's (VF_NO_SPEC=1) on the same rays."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_extra in ({}, {"VF_NO_SPEC": "1"}):
        env = dict(os.environ, ROOT=root, **env_extra)
        env.pop("VF_NO_SPEC", None) if not env_extra else None
        r = subprocess.run([sys.executable, "-c", _COUNT_CHILD, kind, fmt], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
    assert outs[0][0]["cell_tests"] > 0 and outs[0][1]["redescents"] >= 0
