"""The restated host offline stage reproduces the reference's operator.

The reference's operators (tests/golden/fx_*.ptc, and the checksums of the
large cases in tests/golden/*_ref.ptc) were captured from the reference
package itself by tools/make_cases.py.
"""

import numpy as np
import pytest

from conftest import FIXTURES, case_path, golden_path
from paper_1410_5910_b200.cache import read_case
from paper_1410_5910_b200.offline import configs
from paper_1410_5910_b200.offline.assemble import polarized_table, sweep_order
from paper_1410_5910_b200.offline.build import (build_operator, compare_checksums,
                                                 operator_checksums)
from paper_1410_5910_b200.offline.compress import plr_leaves
from paper_1410_5910_b200.offline.layers import equal_partition


def test_media_reproduce_survey_values():
    # c2 c_max 3.837, omega 377.93; c3 c_min 1.8426, c_max 5.325, omega 1159.18
    c2, c3 = configs.config("c2"), configs.config("c3")
    assert c2.c.min() == 1.5 and abs(c2.c.max() - 3.8374584789) < 1e-9
    assert abs(c2.omega - 377.9335962268) < 1e-6
    assert abs(c3.c.min() - 1.8425966686) < 1e-9 and abs(c3.c.max() - 5.3250690193) < 1e-9
    assert abs(c3.omega - 1159.1848035439) < 1e-6
    assert c3.geo.nx_ext == 880 and c2.geo.nx_ext == 460


def test_partition_remainder_to_front():
    # partition.py:68-84 ; fx_uneven is 19 rows in 4 layers
    assert list(np.diff(equal_partition(19, 4))) == [5, 5, 5, 4]
    with pytest.raises(ValueError):
        equal_partition(5, 3)


@pytest.mark.parametrize("name", FIXTURES + ["c1_ref", "c3r_ref", "c2_ref", "c3_ref"])
def test_entry_table_matches_reference(name):
    meta, arr = read_case(golden_path(name))
    entries, coefs, keys, perm = polarized_table(meta["n_c"], meta["h"], meta.get("variant", "jump"))
    assert np.array_equal(entries, arr["entries"])
    assert np.array_equal(coefs, arr["coefs"])
    assert np.array_equal(perm, arr["perm"])
    assert np.array_equal(sweep_order(meta["L"]), arr["perm"])


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_operators_bitwise(name):
    meta, arr = build_operator(name, workers=1)
    rm, ra = read_case(golden_path(name))
    if "dense" in ra:
        assert np.array_equal(arr["dense"], ra["dense"])
    else:
        assert np.array_equal(arr["leaves"], ra["leaves"])
        assert np.array_equal(arr["factors"], ra["factors"])
    assert np.array_equal(arr["rhs"][0], ra["rhs"][0])


def test_c1_operator_matches_reference_checksums():
    meta, arr = build_operator("c1", workers=4)
    rm, ra = read_case(golden_path("c1_ref"))
    compare_checksums(operator_checksums(meta, arr), ra, rtol=1e-12)
    d = np.abs(arr["rhs"][0] - ra["rhs"][0]).max() / np.abs(ra["rhs"][0]).max()
    assert d <= 1e-12


def test_c3r_plr_structure_matches_reference():
    meta, arr = build_operator("c3r", workers=4)
    rm, ra = read_case(golden_path("c3r_ref"))
    compare_checksums(operator_checksums(meta, arr), ra, rtol=1e-12)


def test_checksum_comparison_detects_differences():
    meta, arr = build_operator("fx_plr", workers=1)
    ck = operator_checksums(meta, arr)
    bad = dict(ck)
    bad["ck_leaves"] = ck["ck_leaves"].copy()
    bad["ck_leaves"][0, 5] += 1
    with pytest.raises(ValueError, match="structure"):
        compare_checksums(bad, ck)
    bad = dict(ck)
    bad["ck_norm"] = ck["ck_norm"] * (1 + 1e-6)
    with pytest.raises(ValueError, match="norms"):
        compare_checksums(bad, ck)


def test_plr_leaves_reconstruct_block():
    # plr.py semantics: leaves tile the block, each within epsilon of the original
    rng = np.random.default_rng(3)
    x = np.linspace(0, 1, 97)
    block = np.exp(1j * 30 * np.abs(x[:, None] - x[None, :] + 0.01))
    block += 1e-3 * (rng.standard_normal(block.shape))
    leaves = plr_leaves(block, r_max=6, eps=1e-9)
    dense = np.zeros_like(block)
    cover = np.zeros(block.shape, dtype=int)
    for (r0, c0, u, vt) in leaves:
        dense[r0:r0 + u.shape[0], c0:c0 + vt.shape[1]] += u @ vt
        cover[r0:r0 + u.shape[0], c0:c0 + vt.shape[1]] += 1
    assert cover.max() == 1
    assert np.abs(dense - block).max() <= 1e-8
