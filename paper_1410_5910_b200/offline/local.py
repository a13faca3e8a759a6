"""Per-layer factorizations for the device local solves (host offline).

The reference factors every layer operator with SuperLU (COLAMD column order,
``LocalFactorization``, local_solver.py:21-60) and solves on the host.  For
the device the same layer operator (``layers.layer_operator``) is factored
once with a geometric nested-dissection order of its nze x nxe grid, which
keeps the dependency depth of the triangular solves short (c3 layer: 738
levels and 7.9 M stored entries with 4 x 4 leaf blocks -- 903 levels and
12.1 M with 16 x 16 leaves, 8,421 levels with SuperLU's COLAMD order), and
diagonal pivoting (the layer operators are diagonally dominant enough;
residuals ~1e-13 are checked):

    P A P^T = A',   Pr A' Pc = L U   (SuperLU, permc NATURAL on A')

so  A x = b  is  y = b[q_in],  L w = y,  U z = w,  x = z[q_out]  with
q_in = p[perm_r^-1] and q_out = perm_c[p^-1].  With diagonal pivoting
SuperLU keeps the order (perm_r = perm_c = identity, checked), so every leaf
block and separator of the dissection is a contiguous run of factor rows;
their offsets (``block_ptr``) let the device solve a whole block at once.
"""

from __future__ import annotations

import os
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .configs import config
from .layers import edge_extend, equal_partition, layer_operator

__all__ = ["nd_order", "factor_layer", "build_local", "apply_factors"]


def nd_order(nze, nxe, min_block=4, blocks=False):
    """Geometric nested dissection of the nze x nxe grid (index z * nxe + x):
    split the longer side by a grid line, order both halves, then the line.
    ``blocks=True`` also returns the start offsets of the leaf blocks and
    separators in the order (plus the total), each a contiguous run."""
    out = []
    starts = []
    stack = [(0, nze, 0, nxe, False)]
    # iterative post-order: (region, emitted-children flag)
    while stack:
        z0, z1, x0, x1, done = stack.pop()
        w, hgt = x1 - x0, z1 - z0
        if w <= 0 or hgt <= 0:
            continue
        if w * hgt <= min_block * min_block or (w <= 2 and hgt <= 2):
            starts.append(len(out))
            out.extend(z * nxe + x for z in range(z0, z1) for x in range(x0, x1))
            continue
        if w >= hgt:
            xm = (x0 + x1) // 2
            if done:
                starts.append(len(out))
                out.extend(z * nxe + xm for z in range(z0, z1))
                continue
            stack.append((z0, z1, x0, x1, True))
            stack.append((z0, z1, xm + 1, x1, False))
            stack.append((z0, z1, x0, xm, False))
        else:
            zm = (z0 + z1) // 2
            if done:
                starts.append(len(out))
                out.extend(zm * nxe + x for x in range(x0, x1))
                continue
            stack.append((z0, z1, x0, x1, True))
            stack.append((zm + 1, z1, x0, x1, False))
            stack.append((z0, zm, x0, x1, False))
    p = np.asarray(out, dtype=np.int64)
    if p.size != nze * nxe or np.unique(p).size != p.size:
        raise AssertionError("nested-dissection order is not a permutation")
    if blocks:
        return p, np.asarray(starts + [len(out)], dtype=np.int64)
    return p


# SuperLU diagonal-pivot thresholds tried in order: 0 keeps the nested-dissection
# order (every block a contiguous run, the device's block solve); the Helmholtz /
# PML operators are indefinite, so a factorization whose residual check fails is
# redone with threshold and then full partial pivoting (rows reordered: the
# device falls back to its row-level solve).
PIVOT_THRESHOLDS = (0.0, 0.1, 1.0)
RESIDUAL_TOL = 1e-10


def factor_layer(op, nze, nxe, check=True, thresholds=PIVOT_THRESHOLDS):
    """Factor one layer operator for the device: dict of CSR L, U and the
    composed gathers q_in / q_out (see the module docstring), plus the pivot
    threshold that was used and the residual of a seeded solve."""
    op = sp.csc_matrix(op)
    p, blocks0 = nd_order(nze, nxe, blocks=True)
    a = sp.csc_matrix(op[p][:, p])
    ident = np.arange(a.shape[0])
    rng = np.random.default_rng(0)
    b = rng.standard_normal(op.shape[0]) + 1j * rng.standard_normal(op.shape[0])
    last = None
    for thresh in thresholds:
        try:
            lu = spla.splu(a, permc_spec="NATURAL", diag_pivot_thresh=thresh)
        except RuntimeError as exc:  # exactly singular pivot: pivot harder
            last = f"threshold {thresh}: {exc}"
            continue
        blocks = blocks0
        if not (np.array_equal(lu.perm_r, ident) and np.array_equal(lu.perm_c, ident)):
            blocks = None  # SuperLU reordered: the blocks are no longer contiguous runs
        L, U = lu.L.tocsr(), lu.U.tocsr()
        L.sort_indices()
        U.sort_indices()
        inv_pr = np.argsort(lu.perm_r)
        inv_p = np.argsort(p)
        fac = {"L": L, "U": U, "q_in": p[inv_pr].astype(np.int64),
               "q_out": np.asarray(lu.perm_c, dtype=np.int64)[inv_p], "block_ptr": blocks,
               "pivot_thresh": thresh, "residual": None}
        if not check:
            return fac
        x = apply_factors(fac, b)
        res = float(np.linalg.norm(op @ x - b) / np.linalg.norm(b))
        fac["residual"] = res
        if res < RESIDUAL_TOL:
            return fac
        last = f"threshold {thresh}: residual {res:.2e}"
    raise RuntimeError(f"layer factorization inaccurate at every pivot threshold ({last})")


def apply_factors(fac, b):
    """Host restatement of the device solve (test infrastructure)."""
    y = b[fac["q_in"]]
    w = spla.spsolve_triangular(fac["L"], y, lower=True)
    z = spla.spsolve_triangular(fac["U"], w, lower=False)
    return z[fac["q_out"]]


def _job(args):
    nx, n_layer, h, n_pml, omega, m_tilde = args
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass
    op = layer_operator(nx, n_layer, h, n_pml, omega, m_tilde)
    return factor_layer(op, n_layer + 2 * n_pml, nx + 2 * n_pml)


def build_local(name, workers=None):
    """Device factorizations of every layer of case ``name`` (layer-parallel).
    Returns (layers, geometry dict)."""
    cfg = config(name)
    g, L = cfg.geo, cfg.L
    n_c = equal_partition(g.nz, L)
    m_ext = edge_extend(1.0 / cfg.c**2, g.n_pml)
    jobs = []
    for ell in range(1, L + 1):
        lo = g.n_pml + n_c[ell - 1]
        n_layer = int(n_c[ell] - n_c[ell - 1])
        rows = m_ext[lo:lo + n_layer, :]
        jobs.append((g.nx, n_layer, g.h, g.n_pml, float(cfg.omega), edge_extend(rows, g.n_pml, axis=0)))
    t0 = time.perf_counter()
    workers = workers or min(L, os.cpu_count() or 1)
    if workers > 1:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(min(workers, L)) as pool:
            facs = pool.map(_job, jobs, chunksize=1)
    else:
        facs = [_job(j) for j in jobs]
    geo = {"nx": g.nx, "nz": g.nz, "n_pml": g.n_pml, "h": g.h, "L": L,
           "n_c": [int(v) for v in n_c], "nxe": g.nx_ext, "variant": cfg.variant,
           "factor_seconds": time.perf_counter() - t0}
    for ell, fac in enumerate(facs, start=1):
        fac["n_layer"] = int(n_c[ell] - n_c[ell - 1])
        fac["n_pml"] = g.n_pml
        fac["nze"] = fac["n_layer"] + 2 * g.n_pml
        fac["nxe"] = g.nx_ext
    return facs, geo
