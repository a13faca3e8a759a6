"""The reference-side drop-in route, exercised end to end on the CPU.

A user of the reference keeps its own offline stage and swaps the online
solve: ``paper_1410_5910_b200.solver.offline_assemble`` runs the reference's
``offline_assemble`` (solver.py:132-193), captures ``state.pol`` /
``state.perm`` (capture.py: entry table, shared kernels, PLR leaves recovered
from the reference's own ``PLRSparseForm`` factors) and uploads them with
``DeviceOperator.from_reference``.  Here the upload is a plan-only handle
(PT_DEVICE_HOST: tables built, no GPU), checked against the golden operator
tools/make_cases.py recorded from the same reference run: identical entry
table, coefficients, permutation, kernel bytes and task plans.  Skipped where
the reference package is absent (the GPU box).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import golden_path
from paper_1410_5910_b200 import solver as S
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not (REF / "helmsweep").exists(),
                                reason="reference package not present (build container only)")


@pytest.mark.parametrize("name", ["fx_tiny", "fx_plr", "fx_extrap_plr"])
def test_reference_offline_assemble_uploads_the_golden_operator(name):
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import make_cases as MC
    cfg = MC.config(name)
    grid, L = cfg["grid"], cfg["L"]
    part = MC.make_partition(grid.nz, L)
    model = MC.model_from_c(grid, cfg["c"])
    state = S.offline_assemble(grid, model, part, float(cfg["omega"]), variant=cfg["variant"],
                               factor_method="sparse", compression=cfg["compression"], device="host")
    gm, ga = load_case_arrays(golden_path(name))
    op = state.op
    assert np.array_equal(op.entries, np.asarray(ga["entries"]))
    assert np.array_equal(op.coefs, np.asarray(ga["coefs"]))
    assert np.array_equal(op.perm, np.asarray(ga["perm"]))
    golden = DeviceOperator.from_arrays(gm, ga, device="host")
    assert op.kernel_format == golden.kernel_format and op.n_kernels == golden.n_kernels
    for kind, n_it in (("A", 0), ("M", 2), ("AM", 2), ("S", 0)):
        mine = op.plan_stats(kind, n_it) if n_it else op.plan_stats(kind)
        ref = golden.plan_stats(kind, n_it) if n_it else golden.plan_stats(kind)
        assert mine == ref, (kind, mine, ref)
    assert state.host_state is not None and "upload" in state.stage_seconds
