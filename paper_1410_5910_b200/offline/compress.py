"""Adaptive partitioned-low-rank compression (host offline), restated.

Follows the reference's quadtree (plr.py:200-236, 268-297): a block whose
smaller side is <= 2 r_max becomes a truncated-SVD leaf keeping the singular
values >= epsilon; otherwise it is accepted as a leaf when sigma_{r_max+1} <
epsilon, else split floor-first into quadrants (TL, TR, BL, BR).  Leaves are
returned in preorder -- the slot order of the reference's PLRSparseForm --
with U carrying U*Sigma; rank-0 leaves are dropped, as to_sparse_form does.
"""

from __future__ import annotations

import numpy as np

__all__ = ["plr_leaves", "leaf_table"]


def _svd_leaf(block, eps):
    u, s, vt = np.linalg.svd(block, full_matrices=False)
    r = int(np.count_nonzero(s >= eps))
    return np.ascontiguousarray(u[:, :r] * s[:r]), np.ascontiguousarray(vt[:r, :])


def plr_leaves(block, r_max, eps):
    """[(row_off, col_off, U (rows x r), Vt (r x cols))] in preorder.

    The split rule is the reference's (sigma_{r_max+1}(node) >= eps), evaluated
    without the node's own SVD where a quadrant already decides it: the
    singular values of a submatrix never exceed the matrix's
    (sigma_k(B[I, J]) <= sigma_k(B)), so a quadrant with sigma_{r_max+1} >= eps
    certifies the split -- and that quadrant's singular values are exactly what
    its own decision needs next.  Only nodes no quadrant certifies (the ones
    that end as leaves, mostly) get their own SVD.  Same leaves; the large
    nodes near the root, which always split, cost nothing."""
    block = np.asarray(block, dtype=np.complex128)
    if block.ndim != 2 or block.size == 0:
        raise ValueError("block must be a nonempty 2D array")
    if r_max < 1 or not eps > 0:
        raise ValueError("need r_max >= 1 and epsilon > 0")
    svals = {}

    def sigma(r0, c0, b):  # singular values of the node at (r0, c0), memoised
        key = (r0, c0, b.shape)
        if key not in svals:
            svals[key] = np.linalg.svd(b, compute_uv=False)
        return svals[key]

    def quadrants(r0, c0, b):
        m, k = b.shape
        rs, cs = m // 2, k // 2
        return [(r0, c0, b[:rs, :cs]), (r0, c0 + cs, b[:rs, cs:]),
                (r0 + rs, c0, b[rs:, :cs]), (r0 + rs, c0 + cs, b[rs:, cs:])]

    def splits(r0, c0, b):
        m, k = b.shape
        if min(m, k) <= 2 * r_max:
            return False
        key = (r0, c0, b.shape)
        if key not in svals:
            for q in quadrants(r0, c0, b):
                if min(q[2].shape) > r_max and sigma(*q)[r_max] >= eps:
                    return True
        return bool(sigma(r0, c0, b)[r_max] >= eps)

    out = []
    stack = [(0, 0, block)]
    while stack:
        r0, c0, b = stack.pop()
        if splits(r0, c0, b):
            # push in reverse so the pops come out TL, TR, BL, BR (preorder)
            stack.extend(reversed(quadrants(r0, c0, b)))
            svals.pop((r0, c0, b.shape), None)
            continue
        svals.pop((r0, c0, b.shape), None)
        u, vt = _svd_leaf(b, eps)
        if u.shape[1]:
            out.append((r0, c0, u, vt))
    return out


def leaf_table(kernels_leaves):
    """Pack per-kernel leaf lists (or dense ndarrays) into the pt_leaf table + factor array."""
    rows, chunks, kbytes = [], [], []
    off = 0
    for kid, leaves in enumerate(kernels_leaves):
        if isinstance(leaves, np.ndarray):  # a dense kernel: one full leaf U = K, Vt = I
            m = leaves.shape[0]
            rows.append((kid, 0, 0, m, m, m, off, off + m * m))
            chunks.append(np.ascontiguousarray(leaves, dtype=np.complex128).ravel())
            chunks.append(np.eye(m, dtype=np.complex128).ravel())
            off += 2 * m * m
            kbytes.append(16 * m * m)
            continue
        nb = 0
        for (r0, c0, u, vt) in leaves:
            ml, r = u.shape
            kk = vt.shape[1]
            rows.append((kid, r0, c0, ml, kk, r, off, off + ml * r))
            chunks.append(u.ravel())
            chunks.append(vt.ravel())
            off += ml * r + r * kk
            nb += 16 * r * (ml + kk)
        kbytes.append(nb)
    table = np.asarray(rows, dtype=np.int64).reshape(-1, 8)
    factors = np.concatenate(chunks) if chunks else np.zeros(0, np.complex128)
    return table, factors, np.asarray(kbytes, dtype=np.int64)
