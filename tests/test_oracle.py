"""Pin the CPU oracle against vectors produced by the reference itself.

tests/golden/*.ptc were written by tools/make_cases.py, which ran the
reference package's own offline_assemble / pol.matvec / preconditioner_apply
/ gs_sweep / solve_helmholtz.  These tests check that oracle/ restates that
arithmetic, so the GPU parity tests can use it as the checker.
"""

import numpy as np
import pytest

from conftest import FIXTURES, case_path, golden_path
from oracle import ref_port as O
from paper_1410_5910_b200.operator import load_case_arrays


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def load(name, big=False):
    path = case_path(name) if big else golden_path(name)
    if not path.exists():
        pytest.skip(f"{path} not generated (python tools/make_cases.py {name})")
    meta, arr = load_case_arrays(path)
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    return meta, arr, pol, perm, d, r


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_applies_match_reference(name):
    meta, arr, pol, perm, d, r = load(name)
    px, pu = np.asarray(arr["probe_x"]), np.asarray(arr["probe_u"])
    assert rel(pol.matvec(px), arr["probe_Ax"]) <= 1e-13
    assert rel(O.preconditioner_apply(2, d, r, perm, px), arr["probe_Mx"]) <= 1e-13
    assert rel(O.preconditioner_apply(1, d, r, perm, px), arr["probe_M1x"]) <= 1e-13
    assert rel(O.gs_sweep(d, r, perm, px, pu), arr["probe_sweep"]) <= 1e-13


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_gmres_matches_reference(name):
    meta, arr, pol, perm, d, r = load(name)
    rhs = np.asarray(arr["rhs"][0])
    x, rep = O.gmres_solve(pol.matvec, lambda v: O.preconditioner_apply(2, d, r, perm, v), rhs,
                           rel_tol=meta["gmres_tol"], max_iter=meta["gmres_max_iter"])
    ref = meta["solves"][0]
    assert rep.iterations == ref["iterations"]
    assert rep.flag == ref["flag"]
    hist = np.asarray(arr["ref_hist"][0][: ref["iterations"]])
    assert np.allclose(rep.residual_history, hist, rtol=1e-6, atol=1e-14)
    assert rel(x, arr["ref_x"][0]) <= 1e-10
    nt, m = meta["nt"], meta["m"]
    assert rel(x[: nt * m] + x[nt * m:], arr["ref_traces"][0]) <= 1e-10


@pytest.mark.parametrize("name", FIXTURES)
def test_split_is_exact_permuted_system(name):
    # trace_system.py:499-524 / test_trace_system.py:347-369
    meta, arr, pol, perm, d, r = load(name)
    m, nt = pol.m, pol.n_block_rows // 2
    dim = nt * m
    full = np.zeros((2 * dim, 2 * dim), dtype=np.complex128)
    full[:dim, :dim] = d[0].to_dense()
    full[:dim, dim:] = r[0].to_dense()
    full[dim:, :dim] = r[1].to_dense()
    full[dim:, dim:] = d[1].to_dense()
    rows = (perm[:, None] * m + np.arange(m)[None, :]).ravel()
    assert np.array_equal(full, pol.to_dense()[rows, :])


@pytest.mark.parametrize("name", FIXTURES)
def test_back_substitution_matches_dense(name):
    meta, arr, pol, perm, d, r = load(name)
    rng = np.random.default_rng(61)
    dim = d[0].n_block_rows * d[0].m
    rhs = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    for tri, kind in ((d[0], "lower"), (d[1], "upper")):
        x = O.solve_block_triangular(tri, rhs, kind)
        x_ref = np.linalg.solve(tri.to_dense(), rhs)
        assert np.abs(x - x_ref).max() <= 1e-10 * np.abs(x_ref).max()


@pytest.mark.parametrize("name", FIXTURES)
def test_case_permutation_is_sweep_order(name):
    meta, arr, *_ = load(name)
    assert np.array_equal(arr["perm"], O.sweep_permutation(meta["L"]))


def test_sweep_permutation_known_answer():
    # test_trace_system.py:443-448
    perm = O.sweep_permutation(4)
    assert sorted(perm.tolist()) == list(range(12))
    assert perm[:6].tolist() == [0, 6, 2, 8, 4, 10]
    assert perm[6:].tolist() == [7, 1, 9, 3, 11, 5]


# ---- the reference's GMRES unit tests (test_solver.py:131-191) on the oracle


def test_gmres_identity_breakdown():
    rng = np.random.default_rng(0)
    b = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    x, rep = O.gmres_solve(lambda v: v, lambda v: v, b)
    assert rep.converged and rep.flag == "breakdown" and rep.iterations == 1
    assert np.abs(x - b).max() <= 1e-13 * np.abs(b).max()


def test_gmres_dense_3x3():
    a = np.array([[4.0, 1.0, 0.0], [1.0, 3.0, 1.0], [0.0, 1.0, 2.0]]) + 0.5j * np.eye(3)
    b = np.array([1.0, -2.0, 0.5]) + 1j * np.array([0.0, 1.0, -0.5])
    x, rep = O.gmres_solve(lambda v: a @ v, lambda v: v, b, rel_tol=1e-12)
    assert rep.converged and rep.iterations <= 3
    assert np.abs(x - np.linalg.solve(a, b)).max() <= 1e-12 * 4


def test_gmres_zero_rhs():
    x, rep = O.gmres_solve(lambda v: v, lambda v: v, np.zeros(5, complex))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0)


def test_gmres_stagnation():
    x, rep = O.gmres_solve(lambda v: np.roll(v, 1), lambda v: v, np.eye(50, dtype=complex)[:, 0],
                           rel_tol=1e-12, max_iter=40)
    assert rep.flag == "stagnation" and not rep.converged


def test_gmres_nan():
    with pytest.raises(RuntimeError, match="non-finite"):
        O.gmres_solve(lambda v: np.full_like(v, np.nan), lambda v: v, np.ones(4, complex))


def test_gmres_maxiter():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((30, 30)) + 1j * rng.standard_normal((30, 30))
    b = rng.standard_normal(30) + 0j
    x, rep = O.gmres_solve(lambda v: a @ v, lambda v: v, b, rel_tol=1e-14, max_iter=5)
    assert rep.flag == "maxiter" and not rep.converged and rep.iterations == 5


@pytest.mark.parametrize("name", ["c1", "c3r"])
def test_oracle_large_cases(name):
    meta, arr, pol, perm, d, r = load(name, big=True)
    px = np.asarray(arr["probe_x"])
    assert rel(pol.matvec(px), arr["probe_Ax"]) <= 1e-13
    assert rel(O.preconditioner_apply(2, d, r, perm, px), arr["probe_Mx"]) <= 1e-13
