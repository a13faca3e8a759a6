"""GPU offline stage: interface Green's blocks and their
partitioned-low-rank compression on the device.

The north star keeps the offline stage on the host; this is the "next" row
after the online path.  The reference extracts every layer's interface blocks
with one multi-right-hand-side sparse solve per source depth
(``extract_interface_greens``, local_solver.py:112-135: delta sources 1/h^2 at
depth k, rows of the solution at the four interface depths, times h) and
compresses each block with an adaptive quadtree of truncated SVDs
(``_compress_node`` / ``_truncated_leaf``, plr.py:200-236).  Those two steps
are 93-96% of the reference's offline time.

Here the layer is factored once on the host in the nested-dissection order
the device local solves use (``offline.local.factor_layer``: ``P A P^T = L U``
with the composed gathers ``q_in`` / ``q_out``) and

* the 4 x nxe delta right-hand sides of a layer are solved on the GPU as two
  sparse triangular solves with dense multi-column right-hand sides per source
  depth (cuSPARSE SpSM through ``torch.triangular_solve`` on CSR factors;
  offline plumbing, not the hot path), only the four target rows are kept;
* the quadtree is walked level by level for all blocks of a layer at once:
  the singular values of every node of one shape come from one batched SVD
  (``torch.linalg.svd`` / cuSOLVER), the split rule and the leaf truncation are
  the reference's (sigma_{r_max+1} >= epsilon splits a node whose smaller side
  exceeds 2 r_max; a leaf keeps the singular values >= epsilon; rank-0 leaves
  are dropped; leaves in preorder TL, TR, BL, BR with U carrying U Sigma).

The results equal the host path's up to the rounding of a different
factorization order and SVD driver; tests/test_gpu_offline.py compares them.
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["DeviceLayer", "plr_leaves_gpu"]


def _csr_cuda(a, device):
    a = a.tocsr()
    a.sort_indices()
    return torch.sparse_csr_tensor(
        torch.from_numpy(a.indptr.astype(np.int64)), torch.from_numpy(a.indices.astype(np.int64)),
        torch.from_numpy(np.ascontiguousarray(a.data, dtype=np.complex128)),
        size=a.shape, dtype=torch.complex128, device=device)


class DeviceLayer:
    """One layer's factors on the device: multi-right-hand-side solves.

    ``fac`` is ``offline.local.factor_layer``'s dict (CSR L with its unit
    diagonal stored, CSR U, gathers q_in / q_out)."""

    def __init__(self, fac, nze, nxe, n_layer, n_pml, h, device="cuda"):
        self.nze, self.nxe, self.n_layer, self.n_pml, self.h = nze, nxe, n_layer, n_pml, h
        self.dim = nze * nxe
        self.device = torch.device(device)
        self.L = _csr_cuda(fac["L"], self.device)
        self.U = _csr_cuda(fac["U"], self.device)
        q_in = np.asarray(fac["q_in"], dtype=np.int64)
        inv_in = np.empty_like(q_in)
        inv_in[q_in] = np.arange(q_in.size)
        self.inv_in = torch.from_numpy(inv_in).to(self.device)   # natural index -> factor row
        self.q_out = torch.from_numpy(np.asarray(fac["q_out"], dtype=np.int64)).to(self.device)

    def row(self, depth):
        """Array row of local depth j (depth j lives at n_pml + j - 1)."""
        return self.n_pml + depth - 1

    def solve_columns(self, b_perm):
        """Z with L U Z = B for a dense (dim x k) block already in factor order."""
        w = torch.triangular_solve(b_perm, self.L, upper=False).solution
        return torch.triangular_solve(w, self.U, upper=True).solution

    def greens(self, pairs, chunk=None):
        """{(j, k): G(z_j, z_k)} (device tensors, nxe x nxe complex128) for the
        requested (target, source) depth pairs: per source depth one multi-column
        solve of the delta sources 1/h^2, the target rows times h."""
        nxe, h = self.nxe, self.h
        chunk = nxe if chunk is None else int(chunk)
        out = {}
        cols = torch.arange(nxe, device=self.device)
        for k in sorted({k for (_, k) in pairs}):
            targets = sorted({j for (j, kk) in pairs if kk == k})
            rk = self.row(k)
            blocks = {j: torch.empty((nxe, nxe), dtype=torch.complex128, device=self.device)
                      for j in targets}
            for lo in range(0, nxe, chunk):
                hi = min(nxe, lo + chunk)
                b = torch.zeros((self.dim, hi - lo), dtype=torch.complex128, device=self.device)
                b[self.inv_in[rk * nxe + cols[lo:hi]], cols[: hi - lo]] = 1.0 / h**2
                z = self.solve_columns(b)
                for j in targets:
                    rj = self.row(j)
                    blocks[j][:, lo:hi] = z[self.q_out[rj * nxe:(rj + 1) * nxe], :]
                del b, z
            for j in targets:
                out[(j, k)] = blocks[j] * h
        return out


def plr_leaves_gpu(blocks, r_max, eps):
    """The reference's adaptive quadtree for a list of square/rectangular
    complex128 device blocks at once.  Returns, per block, the host leaf list
    [(row_off, col_off, U Sigma (rows x r), Vt (r x cols))] in preorder, as
    ``offline.compress.plr_leaves`` does.

    Level by level: all open nodes of one shape are stacked and their singular
    values (and vectors, for the nodes that become leaves) come from one
    batched SVD."""
    if r_max < 1 or not eps > 0:
        raise ValueError("need r_max >= 1 and epsilon > 0")
    # node: (block index, path of quadrant digits, r0, c0, view)
    open_nodes = [(i, (), 0, 0, b) for i, b in enumerate(blocks)]
    leaves = [[] for _ in blocks]
    while open_nodes:
        by_shape = {}
        for node in open_nodes:
            by_shape.setdefault(tuple(node[4].shape), []).append(node)
        open_nodes = []
        for (m, k), nodes in by_shape.items():
            stack = torch.stack([n[4] for n in nodes])
            u, s, vt = torch.linalg.svd(stack, full_matrices=False)
            small = min(m, k) <= 2 * r_max
            split = torch.zeros(len(nodes), dtype=torch.bool) if small else (s[:, r_max] >= eps).cpu()
            ranks = (s >= eps).sum(dim=1).cpu()
            us = u * s.unsqueeze(1)
            for idx, (bi, path, r0, c0, blk) in enumerate(nodes):
                if bool(split[idx]):
                    rs, cs = m // 2, k // 2
                    open_nodes.append((bi, path + (0,), r0, c0, blk[:rs, :cs]))
                    open_nodes.append((bi, path + (1,), r0, c0 + cs, blk[:rs, cs:]))
                    open_nodes.append((bi, path + (2,), r0 + rs, c0, blk[rs:, :cs]))
                    open_nodes.append((bi, path + (3,), r0 + rs, c0 + cs, blk[rs:, cs:]))
                    continue
                r = int(ranks[idx])
                if r:
                    leaves[bi].append((path, r0, c0, us[idx, :, :r].cpu().numpy().copy(),
                                       vt[idx, :r, :].cpu().numpy().copy()))
            del u, s, vt, us, stack
    out = []
    for lst in leaves:
        lst.sort(key=lambda t: t[0])  # preorder = lexicographic order of the quadrant paths
        out.append([(r0, c0, np.ascontiguousarray(uu), np.ascontiguousarray(vv))
                    for (_, r0, c0, uu, vv) in lst])
    return out
