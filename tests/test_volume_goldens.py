"""The reference volume-field records (tests/golden/c*_vol.ptc) are usable
checks: present for every BASELINE configuration with a reference solve, of
the reference's shape, and the c3 digest is sensitive to a 1e-8 change.

The records come from tools/make_volume_goldens.py, which runs the
reference's own offline_assemble + solve_helmholtz (solver.py:132-193,
308-435) here; the GPU test is tests/test_gpu_local.py::
test_large_case_volume_matches_reference.
"""

import numpy as np
import pytest

from conftest import golden_path
from paper_1410_5910_b200.operator import load_case_arrays


@pytest.mark.parametrize("name,shape", [("c1", (200, 240)), ("c2", (400, 460)), ("c3", (800, 880))])
def test_volume_record_shapes(name, shape):
    meta, vol = load_case_arrays(golden_path(f"{name}_vol"))
    assert tuple(meta["u_shape"]) == shape
    ref_it = load_case_arrays(golden_path(f"{name}_ref"))[0]["solves"][0]["iterations"]
    assert meta["iterations"] == ref_it
    if "ref_u" in vol:
        assert np.asarray(vol["ref_u"]).shape == shape
        assert np.isfinite(np.asarray(vol["ref_u"])).all()
    else:
        assert np.asarray(vol["ref_u_rows"]).shape[1] == shape[1]
        assert np.asarray(vol["ref_u_proj"]).shape == (16,)


def test_c3_digest_detects_small_changes():
    """A field equal to the recorded rows but perturbed by 1e-7 relative on
    rows the digest does not store is still caught by the projections."""
    from test_gpu_local import volume_error
    meta, vol = load_case_arrays(golden_path("c3_vol"))
    rows = np.asarray(vol["ref_u_row_index"])
    u = np.zeros(tuple(meta["u_shape"]), dtype=np.complex128)
    u[rows] = np.asarray(vol["ref_u_rows"])
    assert volume_error(u, vol) > 1e-3  # unrecorded rows missing: caught
