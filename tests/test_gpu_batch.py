"""GPU parity of the multi-RHS path.

The reference solves many sources one `gmres_solve` after another
(cli.py:380-409).  `pt_gmres_batch` runs up to 64 of them in lockstep on the
batched executor (FP64 tensor-core contractions).  Bars, as for one source:
every apply within 1e-12 relative L2 of the oracle / the reference's own
vectors, per-source iterations within +-1 of the single solve and of the
reference, solutions and traces within 1e-8.
"""

import numpy as np
import pytest

from conftest import FIXTURES
from oracle import ref_port as O
from test_gpu_parity import APPLY_TOL, TRACE_TOL, get, rel

pytestmark = pytest.mark.gpu

DENSE = ["fx_l2", "fx_tiny", "fx_uneven"]
assert set(DENSE) <= set(FIXTURES)


def sources(n, N, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, N)) + 1j * rng.standard_normal((n, N))


@pytest.mark.parametrize("name", DENSE)
@pytest.mark.parametrize("nrhs", [1, 5, 64, 70])
def test_apply_batch_matches_oracle(cuda_ok, name, nrhs):
    meta, arr, op = get(name)
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    X = sources(nrhs, op.N, 100 + nrhs)
    X[0] = arr["probe_x"]
    Y = op.apply_A_batch(X)
    Z = op.apply_M_batch(X, n_it=2)
    Z1 = op.apply_M_batch(X, n_it=1)
    # the reference's own probe vectors
    assert rel(Y[0], arr["probe_Ax"]) <= APPLY_TOL
    assert rel(Z[0], arr["probe_Mx"]) <= APPLY_TOL
    assert rel(Z1[0], arr["probe_M1x"]) <= APPLY_TOL
    for s in range(nrhs):
        assert rel(Y[s], pol.matvec(X[s])) <= APPLY_TOL
        assert rel(Z[s], O.preconditioner_apply(2, d, r, perm, X[s])) <= APPLY_TOL


@pytest.mark.parametrize("name", DENSE)
def test_apply_batch_repeatable_and_column_independent(cuda_ok, name):
    import torch
    meta, arr, op = get(name)
    X = torch.from_numpy(sources(64, op.N, 7)).cuda()
    Y = op.apply_M_batch(X)
    assert torch.equal(Y, op.apply_M_batch(X))
    # a source's result does not depend on the other sources of its batch
    assert torch.equal(op.apply_M_batch(X[:5].contiguous()), Y[:5])
    assert torch.equal(op.apply_A_batch(X[3:4].contiguous()), op.apply_A_batch(X)[3:4])


def _batch_sources(arr, N):
    B = sources(9, N, 5)
    B[0] = arr["rhs"][0]       # the reference's recorded right-hand side
    B[4] = 0.0                 # zero source: x = 0, 0 iterations (solver.py:239-242)
    B[6] = 1e-30 * B[6]        # tiny scale: same iterations as its unscaled self
    return B


@pytest.mark.parametrize("name", DENSE)
def test_gmres_batch_matches_single_and_reference(cuda_ok, name):
    meta, arr, op = get(name)
    tol = meta["gmres_tol"]
    B = _batch_sources(arr, op.N)
    X, reps = op.gmres_batch(B, rel_tol=tol)
    for s in range(B.shape[0]):
        x1, r1 = op.gmres(B[s], rel_tol=tol)
        assert abs(reps[s]["iterations"] - r1["iterations"]) <= 1, s
        assert reps[s]["converged"] == r1["converged"]
        if s == 4:
            assert reps[s]["iterations"] == 0 and reps[s]["converged"]
            assert not np.any(X[s])
            continue
        assert rel(X[s], x1) <= TRACE_TOL
        assert reps[s]["true_residual"] <= 10 * tol
        k = min(reps[s]["iterations"], r1["iterations"])
        assert np.allclose(reps[s]["residual_history"][:k], r1["residual_history"][:k],
                           rtol=1e-6, atol=1e-15)
    # source 0 against the reference's own solve
    ref = meta["solves"][0]
    assert abs(reps[0]["iterations"] - ref["iterations"]) <= 1
    nt, m = meta["nt"], meta["m"]
    assert rel(X[0][: nt * m] + X[0][nt * m:], arr["ref_traces"][0]) <= TRACE_TOL
    # and a random source against the oracle's MGS + lstsq GMRES
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    xo, ro = O.gmres_solve(pol.matvec, lambda v: O.preconditioner_apply(2, d, r, perm, v), B[2],
                           rel_tol=tol)
    assert abs(reps[2]["iterations"] - ro.iterations) <= 1
    assert rel(X[2], xo) <= TRACE_TOL


@pytest.mark.parametrize("name", DENSE[:1])
def test_gmres_batch_host_and_repeatable(cuda_ok, name):
    import torch
    meta, arr, op = get(name)
    tol = meta["gmres_tol"]
    B = _batch_sources(arr, op.N)
    X1, r1 = op.gmres_batch(B, rel_tol=tol)
    X2, r2 = op.gmres_batch(B, rel_tol=tol)
    assert np.array_equal(X1, X2)
    Bh = torch.from_numpy(B).pin_memory()
    Xh = torch.empty_like(Bh).pin_memory()
    rh = op.gmres_batch_host(Bh, Xh, rel_tol=tol)
    assert np.array_equal(Xh.numpy(), X1)
    assert [r["iterations"] for r in rh] == [r["iterations"] for r in r1]


def test_gmres_batch_more_than_one_batch(cuda_ok):
    meta, arr, op = get("fx_l2")
    tol = meta["gmres_tol"]
    B = sources(70, op.N, 9)
    X, reps = op.gmres_batch(B, rel_tol=tol)
    for s in (0, 63, 64, 69):
        x1, r1 = op.gmres(B[s], rel_tol=tol)
        assert abs(reps[s]["iterations"] - r1["iterations"]) <= 1
        assert rel(X[s], x1) <= TRACE_TOL


def test_gmres_batch_nan_source_raises(cuda_ok):
    meta, arr, op = get("fx_tiny")
    B = sources(3, op.N, 4)
    B[1, 3] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        op.gmres_batch(B, rel_tol=meta["gmres_tol"])


def test_gmres_batch_maxiter_per_source(cuda_ok):
    meta, arr, op = get("fx_uneven")
    B = sources(4, op.N, 12)
    X, reps = op.gmres_batch(B, rel_tol=1e-15, max_iter=3)
    for s in range(4):
        x1, r1 = op.gmres(B[s], rel_tol=1e-15, max_iter=3)
        assert reps[s]["iterations"] == r1["iterations"]
        assert reps[s]["flag"] == r1["flag"]


@pytest.mark.slow
def test_c5_batched_parity(cuda_ok):
    meta, arr, op = get("c5", big=True)
    nt, m = meta["nt"], meta["m"]
    B = np.asarray(arr["rhs"])
    assert B.shape[0] == 64
    X, reps = op.gmres_batch(B, rel_tol=meta["gmres_tol"])
    for i, s in enumerate(np.asarray(arr["ref_index"])):
        assert abs(reps[s]["iterations"] - meta["solves"][i]["iterations"]) <= 1
        assert rel(X[s][: nt * m] + X[s][nt * m:], arr["ref_traces"][i]) <= TRACE_TOL
    for r in reps:
        assert r["converged"] and r["true_residual"] <= 10 * meta["gmres_tol"]


@pytest.mark.parametrize("tile", [("PT_BATCH_ROWS", "8"), ("PT_BATCH_ROWS", "16"), ("PT_BATCH_COLS", "32")])
def test_batch_tiles_agree(cuda_ok, tile, monkeypatch):
    """Every batched tile shape (16x32 default, 8x64, 16x64) gives the same
    applies to rounding and the same per-source iterations."""
    from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays
    from conftest import golden_path
    meta, arr = load_case_arrays(golden_path("fx_uneven"))
    monkeypatch.setenv(*tile)
    op = DeviceOperator.from_arrays(meta, arr)  # fresh handle: the tile is read at first use
    X = sources(40, op.N, 21)
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    Z = op.apply_M_batch(X)
    for s in (0, 17, 39):
        assert rel(Z[s], O.preconditioner_apply(2, d, r, perm, X[s])) <= APPLY_TOL
    Xs, reps = op.gmres_batch(X[:6], rel_tol=meta["gmres_tol"])
    for s in range(6):
        x1, r1 = op.gmres(X[s], rel_tol=meta["gmres_tol"])
        assert abs(reps[s]["iterations"] - r1["iterations"]) <= 1
        assert rel(Xs[s], x1) <= TRACE_TOL
    op.close()
