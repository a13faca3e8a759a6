"""GPU parity of the device local solves.

Newton traces -> polarized right-hand side against the reference's own
right-hand side, volume reconstruction against the reference's volume field,
and the whole online pipeline (solve_helmholtz with every stage on the
device) against the reference's field.  Bars: right-hand side 1e-10 (it is a
GMRES input), volume 1e-8 (BASELINE north_star).
"""

import numpy as np
import pytest

from conftest import FIXTURES, golden_path
from paper_1410_5910_b200.offline import configs
from paper_1410_5910_b200.offline.local import apply_factors, build_local
from paper_1410_5910_b200.operator import load_case_arrays
from test_gpu_parity import TRACE_TOL, rel

pytestmark = pytest.mark.gpu

_LOC = {}


def local(name):
    from paper_1410_5910_b200.local import DeviceLocalSolver
    if name not in _LOC:
        facs, geo = build_local(name, workers=1)
        _LOC[name] = (facs, geo, DeviceLocalSolver(facs, geo))
    return _LOC[name]


@pytest.mark.parametrize("name", FIXTURES)
def test_rhs_and_volume_match_reference(cuda_ok, name):
    meta, arr = load_case_arrays(golden_path(name))
    facs, geo, loc = local(name)
    f = configs.config(name).sources[0][1]
    assert rel(loc.rhs(f, meta.get("variant", "jump")), arr["rhs"][0]) <= 1e-10
    u = loc.reconstruct(f, arr["ref_x"][0])
    assert rel(u, arr["ref_u"]) <= TRACE_TOL


@pytest.mark.parametrize("name", ["fx_plr", "fx_uneven"])
def test_layer_solve_matches_host_restatement(cuda_ok, name):
    import torch
    facs, geo, loc = local(name)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(loc.info["rows"]) + 1j * rng.standard_normal(loc.info["rows"])
    x = loc.solve(b)
    off = 0
    for fac in facs:
        n = fac["nze"] * fac["nxe"]
        assert rel(x[off:off + n], apply_factors(fac, b[off:off + n])) <= 1e-12
        off += n
    bd = torch.from_numpy(b).cuda()
    assert torch.equal(loc.solve(bd), loc.solve(bd))  # fixed summation order: repeatable


@pytest.mark.parametrize("name", ["fx_tiny", "fx_plr", "fx_extrap_plr"])
def test_device_pipeline_end_to_end(cuda_ok, name):
    from paper_1410_5910_b200 import solver as S
    meta, arr = load_case_arrays(golden_path(name))
    state = S.OfflineState.from_case(golden_path(name), local=True)
    f = configs.config(name).sources[0][1]
    pc = S.PreconditionerConfig(variant=meta.get("variant", "jump"))
    rep = S.solve_helmholtz(None, None, None, f, state=state, precond=pc,
                            gmres=S.GmresConfig(rel_tol=meta["gmres_tol"]), oracle=arr["ref_u"])
    assert abs(rep.iterations - meta["solves"][0]["iterations"]) <= 1
    assert rel(rep.traces, arr["ref_traces"][0]) <= TRACE_TOL
    assert rep.oracle_rel_error <= TRACE_TOL
    assert set(rep.stage_seconds) >= {"restrict", "rhs", "gmres", "reconstruct"}
    # zero source: x = 0, u = 0 (solver.py:378-380)
    z = S.solve_helmholtz(None, None, None, np.zeros_like(f), state=state, precond=pc)
    assert z.iterations == 0 and z.converged and not np.any(z.u)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_large_case_rhs_matches_reference(cuda_ok, name):
    from paper_1410_5910_b200.local import DeviceLocalSolver
    meta, arr = load_case_arrays(golden_path(f"{name}_ref"))
    loc = DeviceLocalSolver.from_config(name)
    f = configs.config(name).sources[0][1]
    assert rel(loc.rhs(f), arr["rhs"][0]) <= 1e-10
    loc.close()


def test_block_and_row_solves_agree(cuda_ok, monkeypatch):
    """The block solve (dissection blocks through their diagonal-block
    inverses) and the row-at-a-time solve give the same layer solutions."""
    from paper_1410_5910_b200.local import DeviceLocalSolver
    facs, geo, loc = local("fx_plr")
    assert loc.info["blocked"]
    monkeypatch.setenv("PT_TRSV_BLOCK", "0")
    rows = DeviceLocalSolver(facs, geo)
    rng = np.random.default_rng(8)
    b = rng.standard_normal(loc.info["rows"]) + 1j * rng.standard_normal(loc.info["rows"])
    assert rel(loc.solve(b), rows.solve(b)) <= 1e-12
    assert rows.info["l_levels"] > loc.info["l_levels"]  # row levels vs block levels
    rows.close()


@pytest.mark.parametrize("case", ["fx_plr", "c1"])
def test_warp_prefix_solve_agrees(cuda_ok, monkeypatch, case):
    """The optional warp-per-block path for the small lower levels
    (PT_TRSV_WARP=1) gives the same layer solutions as the CTA-per-block
    solve (c1 has levels with blocks above 32 rows: the prefix ends there
    and the CTA kernel takes the rest)."""
    from paper_1410_5910_b200.local import DeviceLocalSolver
    if case.startswith("fx_"):
        facs, geo, loc = local(case)
        make = lambda: DeviceLocalSolver(facs, geo)  # noqa: E731
    else:
        loc = DeviceLocalSolver.from_config(case)
        make = lambda: DeviceLocalSolver.from_config(case)  # noqa: E731
    monkeypatch.setenv("PT_TRSV_WARP", "1")
    warp = make()
    rng = np.random.default_rng(9)
    b = rng.standard_normal(loc.info["rows"]) + 1j * rng.standard_normal(loc.info["rows"])
    assert rel(loc.solve(b), warp.solve(b)) <= 1e-12
    warp.close()
    if not case.startswith("fx_"):
        loc.close()


def volume_error(u, vol):
    """Relative error of a volume field against the reference's record
    (tools/make_volume_goldens.py): the full field, or for c3 every recorded
    grid row, the norm and 16 seeded projections."""
    if "ref_u" in vol:
        return rel(u, np.asarray(vol["ref_u"]))
    rows = np.asarray(vol["ref_u_row_index"])
    ref_rows = np.asarray(vol["ref_u_rows"])
    nrm = float(np.asarray(vol["ref_u_norm"])[0])
    errs = [rel(u[rows], ref_rows), abs(np.linalg.norm(u) - nrm) / nrm]
    from volume_digest import projections  # the generator's own vectors
    for p, ref in zip(projections(u.shape), np.asarray(vol["ref_u_proj"])):
        errs.append(abs(np.vdot(p, u) - ref) / (np.linalg.norm(p) * nrm))
    return max(errs)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_large_case_volume_matches_reference(cuda_ok, name):
    """North-star bar at the BASELINE configurations: the volume field of the
    whole device online stage (Newton traces, rhs, GMRES, reconstruction)
    within 1e-8 of the reference's own solve_helmholtz (report.u,
    local_solver.py:147-176), and the iteration count within +-1."""
    from paper_1410_5910_b200 import solver as S
    from paper_1410_5910_b200.offline.build import ensure_case
    vmeta, vol = load_case_arrays(golden_path(f"{name}_vol"))
    path = ensure_case(name)
    meta, _ = load_case_arrays(path)
    state = S.OfflineState.from_case(path, local=True)
    f = configs.config(name).sources[0][1]
    rep = S.solve_helmholtz(None, None, None, f, state=state,
                            precond=S.PreconditionerConfig(variant=meta.get("variant", "jump")),
                            gmres=S.GmresConfig(rel_tol=meta["gmres_tol"]))
    assert abs(rep.iterations - vmeta["iterations"]) <= 1
    assert tuple(rep.u.shape) == tuple(vmeta["u_shape"])
    assert volume_error(rep.u, vol) <= TRACE_TOL
    state.local.close()
