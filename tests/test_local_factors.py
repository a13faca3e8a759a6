"""Host side of the device local solves, no GPU.

The nested-dissection factorization of every layer (offline/local.py) must
solve the reference's layer systems: the composed gathers q_in / q_out and the
triangular factors, applied on the host exactly as the device applies them,
reproduce the Newton traces behind the reference's polarized right-hand side
(tests/golden fixtures) and the reference's volume field.
"""

import numpy as np
import pytest

from conftest import FIXTURES, golden_path
from paper_1410_5910_b200.cache import read_case
from paper_1410_5910_b200.offline import configs
from paper_1410_5910_b200.offline.assemble import polarized_rhs
from paper_1410_5910_b200.offline.layers import edge_extend, equal_partition, layer_operator
from paper_1410_5910_b200.offline.local import apply_factors, build_local, factor_layer, nd_order


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_nd_order_is_a_permutation():
    for nze, nxe in ((7, 9), (30, 50), (1, 5), (16, 16), (40, 3)):
        p = nd_order(nze, nxe)
        assert np.array_equal(np.sort(p), np.arange(nze * nxe))


def _layer_fields(name, facs, geo, f):
    """Newton traces and polarized rhs (jump/extrapolation) on the host."""
    newtons = []
    nxe, n_pml = geo["nxe"], geo["n_pml"]
    for ell, fac in enumerate(facs, start=1):
        n = fac["n_layer"]
        lo = n_pml + geo["n_c"][ell - 1]
        fl = np.zeros((fac["nze"], nxe), dtype=np.complex128)
        fl[n_pml:n_pml + n] = f[lo:lo + n]
        w = apply_factors(fac, fl.ravel()).reshape(fac["nze"], nxe)
        newtons.append({k: w[n_pml + k - 1] for k in (0, 1, n, n + 1)})
    return newtons


@pytest.mark.parametrize("name", FIXTURES)
def test_host_restatement_matches_reference_rhs(name):
    meta, arr = read_case(golden_path(name))
    facs, geo = build_local(name, workers=1)
    cfg = configs.config(name)
    newtons = _layer_fields(name, facs, geo, cfg.sources[0][1])
    rhs = polarized_rhs(newtons, geo["n_c"], meta.get("variant", "jump"))
    assert rel(rhs, arr["rhs"][0]) <= 1e-10


def test_factor_layer_residual_and_levels():
    cfg = configs.config("fx_plr")
    g = cfg.geo
    n_c = equal_partition(g.nz, cfg.L)
    m_ext = edge_extend(1.0 / cfg.c**2, g.n_pml)
    lo = g.n_pml + n_c[1]
    n_layer = int(n_c[2] - n_c[1])
    op = layer_operator(g.nx, n_layer, g.h, g.n_pml, float(cfg.omega),
                        edge_extend(m_ext[lo:lo + n_layer], g.n_pml, axis=0))
    fac = factor_layer(op, n_layer + 2 * g.n_pml, g.nx_ext)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(op.shape[0]) + 1j * rng.standard_normal(op.shape[0])
    assert np.linalg.norm(op @ apply_factors(fac, b) - b) <= 1e-12 * np.linalg.norm(b)
    assert np.allclose(fac["L"].diagonal(), 1.0)


def test_nd_blocks_are_contiguous_runs_of_the_factor():
    """The dissection blocks handed to the device: contiguous, covering, and
    SuperLU kept the order (so each block's diagonal block is triangular)."""
    p, starts = nd_order(12, 40, blocks=True)
    assert starts[0] == 0 and starts[-1] == p.size and np.all(np.diff(starts) > 0)
    facs, geo = build_local("fx_plr", workers=1)
    for fac in facs:
        bp = fac["block_ptr"]
        assert bp is not None and bp[-1] == fac["L"].shape[0]
        # no entry of L couples a row to a LATER block (lower triangular by blocks)
        L = fac["L"].tocoo()
        blk = np.searchsorted(bp, np.arange(L.shape[0]), side="right") - 1
        assert np.all(blk[L.col] <= blk[L.row])


def test_pivoting_fallback_on_an_unstable_diagonal():
    """Helmholtz/PML layer operators are indefinite: when the diagonal-pivot
    (nested-dissection preserving) factorization fails its residual check,
    factor_layer redoes it with threshold / partial pivoting and reports the
    threshold and residual; the device then uses the row-level solve
    (block_ptr None when rows were reordered)."""
    import scipy.sparse as sp
    n = 4 * 5
    rng = np.random.default_rng(11)
    # tiny diagonal, O(1) couplings: the unpivoted elimination blows up
    a = sp.random(n, n, density=0.3, random_state=3, format="csc") * 1.0
    a = a + sp.diags(np.full(n, 1e-13)) + sp.diags(np.ones(n - 1), 1) + sp.diags(np.ones(n - 1), -1)
    a = sp.csc_matrix(a.astype(np.complex128))
    fac = factor_layer(a, 4, 5)
    assert fac["residual"] < 1e-10
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert np.linalg.norm(a @ apply_factors(fac, b) - b) <= 1e-10 * np.linalg.norm(b)
    # the nested-dissection-preserving pass alone is rejected loudly
    with pytest.raises(RuntimeError):
        factor_layer(a, 4, 5, thresholds=(0.0,))


def test_regular_layers_keep_the_dissection_order():
    facs, geo = build_local("fx_plr", workers=1)
    assert all(f["pivot_thresh"] == 0.0 and f["residual"] < 1e-10 for f in facs)
