"""Flatten a reference offline state into the upload tables of ``pt_create``.

Works by duck typing on the reference objects (no import of the reference):
``state.pol`` is a ``BlockInterfaceMatrix`` whose ``entries`` map
(block row, block col) -> ``BlockEntry`` (kernel, scale, eye)
(trace_system.py:145-226); kernels are shared by reference between entries
(trace_system.py:388-395) and are either dense ndarrays or
``PLRSparseForm`` objects (plr.py:239-297).  PLR leaves are recovered from
the reference's own sparse factors so the device streams exactly the bytes
the reference multiplies with.
"""

from __future__ import annotations

import numpy as np

__all__ = ["capture_operator", "leaves_from_sparse_form"]


def leaves_from_sparse_form(sf):
    """Recover the quadtree leaves of a PLRSparseForm (plr.py:268-297).

    ``to_sparse_form`` assigns slots leaf by leaf in preorder; one leaf owns a
    run of consecutive slots that share a row range (column of ``left``) and
    a column range (row of ``right``).  Explicit zeros are stored, so the
    ranges are exact.  Returns [(row_off, col_off, U (rows x r), Vt (r x cols))].
    """
    left = sf.left.tocsc()
    right = sf.right.tocsr()
    n_slots = right.shape[0]
    spans = []
    for s in range(n_slots):
        rows = left.indices[left.indptr[s]:left.indptr[s + 1]]
        cols = right.indices[right.indptr[s]:right.indptr[s + 1]]
        spans.append((int(rows.min()), int(rows.max()) + 1, int(cols.min()), int(cols.max()) + 1))
    leaves = []
    s = 0
    while s < n_slots:
        e = s + 1
        while e < n_slots and spans[e] == spans[s]:
            e += 1
        r0, r1, c0, c1 = spans[s]
        if left.indptr[s + 1] - left.indptr[s] != r1 - r0 or \
                right.indptr[s + 1] - right.indptr[s] != c1 - c0:
            raise ValueError("PLR sparse form is not a leaf-contiguous factor pair")
        u = sf.left[r0:r1, s:e].toarray()
        vt = sf.right[s:e, c0:c1].toarray()
        leaves.append((r0, c0, u, vt))
        s = e
    return leaves


def capture_operator(pol, perm, check=True):
    """Return (meta, arrays) for ``pol`` (BlockInterfaceMatrix) and ``perm``.

    arrays: entries (E,3) int64 [row, col, kernel|-1], coefs (E,2) complex
    [scale, eye], perm, kernel_bytes, and either ``dense`` (K,m,m) or
    ``leaves`` (n,8) int64 [kernel,row_off,col_off,rows,cols,rank,u_off,vt_off]
    + ``factors`` (complex; U row-major then Vt row-major per leaf).
    """
    m = pol.m
    items = sorted(pol.entries.items())
    kid, kernels = {}, []
    entries = np.zeros((len(items), 3), dtype=np.int64)
    coefs = np.zeros((len(items), 2), dtype=np.complex128)
    for n, ((i, j), e) in enumerate(items):
        k = -1
        if e.kernel is not None:
            key = id(e.kernel)
            if key not in kid:
                kid[key] = len(kernels)
                kernels.append(e.kernel)
            k = kid[key]
        entries[n] = (i, j, k)
        coefs[n] = (e.scale, e.eye)
    arrays = {"entries": entries, "coefs": coefs, "perm": np.asarray(perm, dtype=np.int64)}
    meta = {"m": int(m), "n_block_rows": int(pol.n_block_rows), "n_kernels": len(kernels)}
    if all(isinstance(k, np.ndarray) for k in kernels):
        meta["kernel_format"] = "dense"
        arrays["dense"] = (np.stack([np.asarray(k, dtype=np.complex128) for k in kernels])
                           if kernels else np.zeros((0, m, m), np.complex128))
        kbytes = [16 * m * m] * len(kernels)
    else:
        meta["kernel_format"] = "plr"
        leaf_rows, chunks, kbytes = [], [], []
        off = 0
        for k_id, sf in enumerate(kernels):
            if isinstance(sf, np.ndarray):
                # a dense kernel next to compressed ones (the extrapolation
                # variant's E blocks, trace_system.py:460-464, are never
                # compressed): one full leaf U = K, Vt = I; the reference
                # reads its m x m entries
                k_arr = np.asarray(sf, dtype=np.complex128)
                leaf_rows.append((k_id, 0, 0, m, m, m, off, off + m * m))
                chunks.append(np.ascontiguousarray(k_arr).ravel())
                chunks.append(np.eye(m, dtype=np.complex128).ravel())
                off += 2 * m * m
                kbytes.append(16 * m * m)
                continue
            leaves = leaves_from_sparse_form(sf)
            nb = 0
            for (r0, c0, u, vt) in leaves:
                ml, r = u.shape
                kk = vt.shape[1]
                leaf_rows.append((k_id, r0, c0, ml, kk, r, off, off + ml * r))
                chunks.append(np.ascontiguousarray(u).ravel())
                chunks.append(np.ascontiguousarray(vt).ravel())
                off += ml * r + r * kk
                nb += 16 * r * (ml + kk)
            if check:
                if nb != 16 * sf.stored_entries():
                    raise ValueError("recovered PLR leaves do not match the stored entries")
                dense = np.zeros((m, m), dtype=np.complex128)
                for (r0, c0, u, vt) in leaves:
                    dense[r0:r0 + u.shape[0], c0:c0 + vt.shape[1]] += u @ vt
                ref = sf.to_dense()
                if np.abs(dense - ref).max() > 1e-12 * max(np.abs(ref).max(), 1e-300):
                    raise ValueError("recovered PLR leaves do not reproduce the factor product")
            kbytes.append(nb)
        arrays["leaves"] = np.asarray(leaf_rows, dtype=np.int64).reshape(-1, 8)
        arrays["factors"] = np.concatenate(chunks) if chunks else np.zeros(0, np.complex128)
    arrays["kernel_bytes"] = np.asarray(kbytes, dtype=np.int64)
    meta["kernel_bytes"] = int(sum(kbytes))
    return meta, arrays
