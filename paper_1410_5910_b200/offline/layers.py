"""Per-layer host work of the offline stage, restated from the reference.

This is host code that the north star keeps on the CPU (the reference's own
offline stage); it is restated here only because the reference package does
not exist on the GPU box, and operator caches above 512 MiB cannot be
shipped there.  Each step follows the reference arithmetic so the operator
matches the reference's up to floating-point rounding (checked against the
reference's checksums, tests/test_offline.py):

* PML stretching  s(x) = (C/d) ((min(x,0)/d)^2 + (max(x-X,0)/d)^2),
  alpha = 1 / (1 + i s / omega), C = 40 ln 10, d = n_pml h   (grid.py:36-77)
* 5-point operator with half-point stretch products, x-fastest ordering,
  Dirichlet neighbours eliminated                          (grid.py:192-269)
* a layer's slowness is its rows edge-extended into the PML (partition.py:116-122)
* sparse LU (SuperLU via scipy splu), solves in 128-column chunks
                                                            (local_solver.py:35-80)
* Green's block G(j,k) = rows of the solve for delta sources 1/h^2 at depth
  k, times h                                                (local_solver.py:112-135)
* Newton traces: one solve of the layer source, four rows  (local_solver.py:138-144)
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

PML_C = 40.0 * math.log(10.0)
SOLVE_CHUNK = 128

__all__ = ["PML_C", "layer_operator", "Layer", "edge_extend", "equal_partition"]


def _stretch(coord, extent, delta, omega, C=PML_C):
    x = np.asarray(coord, dtype=np.float64)
    below = np.minimum(x, 0.0)
    above = np.maximum(x - extent, 0.0)
    s = (C / delta) * ((below / delta) ** 2 + (above / delta) ** 2)
    return np.where(s == 0.0, 1.0 + 0.0j, 1.0 / (1.0 + 1j * s / omega))


def layer_operator(nx, n_rows, h, n_pml, omega, m_ext, C=PML_C):
    """CSR Helmholtz operator on an (n_rows + 2 n_pml) x (nx + 2 n_pml) box."""
    nxe, nze = nx + 2 * n_pml, n_rows + 2 * n_pml
    if m_ext.shape != (nze, nxe):
        raise ValueError(f"slowness extent {m_ext.shape} != extended grid {(nze, nxe)}")
    delta = n_pml * h
    lx, lz = (nx + 1) * h, (n_rows + 1) * h
    ax = _stretch(np.arange(-n_pml + 1, nx + n_pml + 1, dtype=np.float64) * h, lx, delta, omega, C)
    az = _stretch(np.arange(-n_pml + 1, n_rows + n_pml + 1, dtype=np.float64) * h, lz, delta,
                  omega, C)
    axh = _stretch((np.arange(-n_pml, nx + n_pml + 1) + 0.5) * h, lx, delta, omega, C)
    azh = _stretch((np.arange(-n_pml, n_rows + n_pml + 1) + 0.5) * h, lz, delta, omega, C)
    w = 1.0 / h**2
    xl, xr = ax * axh[:-1] * w, ax * axh[1:] * w   # couplings to ix-1 / ix+1
    zl, zr = az * azh[:-1] * w, az * azh[1:] * w   # couplings to iz-1 / iz+1
    centre = ((xl + xr)[np.newaxis, :] + (zl + zr)[:, np.newaxis]
              - omega**2 * m_ext).astype(np.complex128)
    idx = np.arange(nze * nxe).reshape(nze, nxe)
    rows = [idx.ravel(), idx[:, 1:].ravel(), idx[:, :-1].ravel(), idx[1:, :].ravel(),
            idx[:-1, :].ravel()]
    cols = [idx.ravel(), (idx[:, 1:] - 1).ravel(), (idx[:, :-1] + 1).ravel(),
            (idx[1:, :] - nxe).ravel(), (idx[:-1, :] + nxe).ravel()]
    vals = [centre.ravel(),
            np.broadcast_to(-xl[np.newaxis, :], (nze, nxe))[:, 1:].ravel(),
            np.broadcast_to(-xr[np.newaxis, :], (nze, nxe))[:, :-1].ravel(),
            np.broadcast_to(-zl[:, np.newaxis], (nze, nxe))[1:, :].ravel(),
            np.broadcast_to(-zr[:, np.newaxis], (nze, nxe))[:-1, :].ravel()]
    dim = nze * nxe
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(dim, dim)).tocsr()


def edge_extend(a, n_pml, axis=None):
    """Replicate the nearest interior value into the pads."""
    if axis is None:
        return np.pad(a, n_pml, mode="edge")
    pad = [(0, 0)] * a.ndim
    pad[axis] = (n_pml, n_pml)
    return np.pad(a, pad, mode="edge")


def equal_partition(nz, L):
    if nz < 2 * L:
        raise ValueError(f"infeasible partition: nz={nz} < 2L={2 * L}")
    base, rem = divmod(nz, L)
    thick = [base + 1 if ell < rem else base for ell in range(L)]
    return np.concatenate([[0], np.cumsum(thick)]).astype(int)


class Layer:
    """One layer: factorised operator and its interface solves."""

    def __init__(self, nx, n_layer, h, n_pml, omega, m_tilde):
        self.n_layer, self.n_pml, self.h = n_layer, n_pml, h
        self.nxe = nx + 2 * n_pml
        self.nze = n_layer + 2 * n_pml
        self.dim = self.nxe * self.nze
        op = layer_operator(nx, n_layer, h, n_pml, omega, m_tilde)
        self.lu = spla.splu(sp.csc_matrix(op))

    def row(self, depth):
        """Array row of local depth j (depth j lives at n_pml + j - 1)."""
        return self.n_pml + depth - 1

    def _solve_chunk(self, rhs):
        chunk = np.asfortranarray(rhs, dtype=np.complex128)
        return self.lu.solve(np.ascontiguousarray(chunk)).reshape(self.dim, -1)

    def solve(self, b):
        single = b.ndim == 1
        rhs = b.reshape(self.dim, -1)
        out = np.empty_like(rhs, dtype=np.complex128)
        for lo in range(0, rhs.shape[1], SOLVE_CHUNK):
            out[:, lo:lo + SOLVE_CHUNK] = self._solve_chunk(rhs[:, lo:lo + SOLVE_CHUNK])
        return out[:, 0] if single else out

    def greens(self, pairs):
        """{(j, k): G(z_j, z_k)} for the requested (target, source) depth pairs.

        Per source depth the delta right-hand sides are solved in the same
        128-column chunks as the reference; only the target rows are kept.
        """
        nxe, h = self.nxe, self.h
        out = {}
        for k in sorted({k for (_, k) in pairs}):
            targets = sorted({j for (j, kk) in pairs if kk == k})
            blocks = {j: np.empty((nxe, nxe), dtype=np.complex128) for j in targets}
            rk = self.row(k)
            for lo in range(0, nxe, SOLVE_CHUNK):
                hi = min(nxe, lo + SOLVE_CHUNK)
                rhs = np.zeros((self.dim, hi - lo), dtype=np.complex128)
                rhs[rk * nxe + np.arange(lo, hi), np.arange(hi - lo)] = 1.0 / h**2
                x = self._solve_chunk(rhs)
                for j in targets:
                    rj = self.row(j)
                    blocks[j][:, lo:hi] = x[rj * nxe:(rj + 1) * nxe, :]
            for j in targets:
                out[(j, k)] = blocks[j] * h
        return out

    def newton(self, f_local):
        """Interface rows {0, 1, n, n+1} of the layer solve with source f_local."""
        w = self.solve(f_local.astype(np.complex128, copy=False).ravel()).reshape(self.nze, self.nxe)
        n = self.n_layer
        return {k: w[self.row(k), :].copy() for k in (0, 1, n, n + 1)}
