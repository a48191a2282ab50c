"""Format signatures through the C ABI (no GPU needed): parser, canonical text, resolutions,
validation rules. Pins: PAPER.md Table 2 (tests/golden/table2_formats.txt) and the §3.2 example."""
from __future__ import annotations

import os

import pytest

from paper_2410_14128_b200 import vf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table2_formats.txt")


def table2():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        label, res, sig = line.strip().split(" ", 2)
        rows.append((int(label), int(res), sig))
    return rows


def test_table2_all_40_parse_with_printed_resolution():
    rows = table2()
    assert len(rows) == 40 and [r[0] for r in rows] == list(range(1, 41))
    for label, res, sig in rows:
        L = vf.parse_format(sig)
        assert vf.format_resolution(L) == (res, res, res), (label, sig)
        # canonical text round-trips
        assert vf.format_to_string(vf.parse_format(vf.format_to_string(L))) == vf.format_to_string(L)


def test_section_3_2_example():
    # "R(1, 0, 2) R(2, 2, 2)---each voxel in the upper level 2 x 1 x 4 grid points to
    # a sub-volume grid of size 4 x 4 x 4"
    assert vf.format_resolution(vf.parse_format("R(1, 0, 2) R(2, 2, 2)")) == (8, 4, 16)
    # "R(1, 0, 2) D(2, 2, 2, 4)"
    L = vf.parse_format("R(1, 0, 2) D(2, 2, 2, 4)")
    assert L[1].kind == vf.VF_DF and L[1].df_max == 4
    assert vf.format_to_string(L) == "R(1, 0, 2) D(2, 2, 2, 4)"


def test_figure_3_example():
    # PAPER.md:140 fig:metaprogramming_system: compile "R(4, 4, 4) G(8)"
    L = vf.parse_format("R(4, 4, 4) G(8)")
    assert vf.format_to_string(L) == "R(4, 4, 4) G(8)" and vf.format_resolution(L) == (4096,) * 3


@pytest.mark.parametrize("sig,status", [
    ("R(1,2)", vf.VF_ERR_PARSE), ("Q(3)", vf.VF_ERR_PARSE), ("", vf.VF_ERR_PARSE), ("G(3", vf.VF_ERR_PARSE),
    ("S(3^3)", vf.VF_ERR_PARSE), ("R(-1,2,3)", vf.VF_ERR_PARSE),
])
def test_parse_errors(sig, status):
    with pytest.raises(vf.VfError) as e:
        vf.parse_format(sig)
    assert e.value.status == status


@pytest.mark.parametrize("sig", [
    "R(2, 2, 2) R(1, 2, 1)",      # non-first level not cubic
    "R(1^3) D(1, 2, 1, 3)",       # same for DF
    "G(0)", "S(0)", "T(3, 1)", "T(2, 0)", "D(2^3, 0)",
    "R(13, 0, 0)",                # > 4096
    "G(7) G(7)",                  # 2^14 > 4096
    "G(12) S(5)",                 # > 16 tiers
])
def test_format_validation_errors(sig):
    with pytest.raises(vf.VfError) as e:
        vf.format_resolution(vf.parse_format(sig))
    assert e.value.status == vf.VF_ERR_FORMAT


def test_baseline_notation():
    # SURVEY.md §8(c) reading A16 (BASELINE.json configs)
    assert vf.signature_from_baseline("SVDAG->Raw<8>", 256) == "G(5) R(3, 3, 3)"
    assert vf.signature_from_baseline("SVO->Raw<32>", 1024) == "S(5) R(5, 5, 5)"
    assert vf.signature_from_baseline("N^3-tree<4>[2]->N^3-tree<4>->Raw<16>", 1024) == "T(2, 2) T(2, 1) R(4, 4, 4)"
    assert vf.signature_from_baseline("SVDAG", 256) == "G(8)"


def test_library_exports_every_declared_symbol():
    import re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "vf.h")).read()
    declared = set(re.findall(r"VF_API\s+[\w\s\*]+?\b(vf_\w+)\s*\(", hdr))
    assert declared == set(vf.EXPORTED), declared ^ set(vf.EXPORTED)
    for name in declared:
        assert hasattr(vf._lib, name)


@pytest.mark.gpu
def test_every_sweep_format_is_compiled_in():
    """Every format of the bench sweeps (cfg1-cfg5, cfg4i, t512 = PAPER.md Table 2 rows 1-40) runs a
    kernel with the format compiled in (the paper's per-format generated code, §4, as a
    template instance), not the generic tier-table kernel (vf_stats.compiled_in)."""
    import bench
    import torch
    from paper_2410_14128_b200 import vf
    keys = torch.tensor([1 | (2 << 21) | (3 << 42)], dtype=torch.int64, device="cuda")
    rgba = torch.tensor([0x01020304], dtype=torch.int32, device="cuda")
    missing = []
    for cfg, fmts in bench.SWEEP.items():
        for fmt in fmts:
            R = vf.format_resolution(vf.parse_format(fmt))
            h = vf.build((keys, rgba, tuple(R)), fmt)
            if not h.stats()["compiled_in"]:
                missing.append(f"{cfg}: {h.signature}")
            h.close()
    assert not missing, missing
