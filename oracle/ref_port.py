"""numpy/scipy restatement of the reference's online path (TEST INFRASTRUCTURE).

Each function names the reference code it restates (pkg/src/helmsweep/).
The arithmetic is the reference's: dense blocks multiply with numpy ``@``
(OpenBLAS zgemv), compressed blocks with two scipy CSR products built the
way ``to_sparse_form`` builds them, GMRES is modified Gram-Schmidt with a
``numpy.linalg.lstsq`` solve every iteration.  Third-party arithmetic lives
in numpy 2.3 / OpenBLAS 0.3.30 and scipy 1.18 (unpinned by the reference,
pyproject.toml:9-12); parity is anchored on golden vectors made by the
reference itself (tests/golden).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

__all__ = [
    "Block", "BlockMatrix", "SparsePair", "operator_from_case", "sweep_permutation",
    "split_dr", "solve_block_triangular", "gs_sweep", "preconditioner_apply",
    "gmres_solve", "OracleReport",
]

STAGNATION_WINDOW = 10
STAGNATION_IMPROVEMENT = 1e-3


class Block:
    """scale * kernel + eye * I  (BlockEntry, trace_system.py:145-180)."""

    __slots__ = ("kernel", "scale", "eye")

    def __init__(self, kernel, scale, eye):
        self.kernel, self.scale, self.eye = kernel, complex(scale), complex(eye)

    def apply(self, x):  # trace_system.py:159-168
        if self.kernel is None:
            y = np.zeros_like(x, dtype=np.complex128)
        elif isinstance(self.kernel, np.ndarray):
            y = self.scale * (self.kernel @ x)
        else:
            y = self.scale * self.kernel.matvec(x)
        if self.eye != 0:
            y = y + self.eye * x
        return y

    def dense(self, m):  # trace_system.py:170-177
        out = np.zeros((m, m), dtype=np.complex128)
        if self.kernel is not None:
            k = self.kernel if isinstance(self.kernel, np.ndarray) else self.kernel.to_dense()
            out += self.scale * k
        if self.eye != 0:
            out[np.diag_indices(m)] += self.eye
        return out


class BlockMatrix:
    """(block row, block col) -> Block  (BlockInterfaceMatrix, trace_system.py:183-239)."""

    def __init__(self, nbr, nbc, m):
        self.n_block_rows, self.n_block_cols, self.m = nbr, nbc, m
        self.entries = {}

    def matvec(self, x):  # trace_system.py:219-226
        m = self.m
        if x.shape != (self.n_block_cols * m,):
            raise ValueError("vector length does not match the block layout")
        y = np.zeros(self.n_block_rows * m, dtype=np.complex128)
        for (i, j), e in self.entries.items():
            y[i * m:(i + 1) * m] += e.apply(x[j * m:(j + 1) * m])
        return y

    def rows(self):  # trace_system.py:212-217
        out = [[] for _ in range(self.n_block_rows)]
        for (i, j), e in sorted(self.entries.items()):
            out[i].append((j, e))
        return out

    def to_dense(self):
        m = self.m
        out = np.zeros((self.n_block_rows * m, self.n_block_cols * m), dtype=np.complex128)
        for (i, j), e in self.entries.items():
            out[i * m:(i + 1) * m, j * m:(j + 1) * m] = e.dense(m)
        return out


class SparsePair:
    """left @ (right @ x) over quadtree leaves (PLRSparseForm, plr.py:239-297)."""

    def __init__(self, m, leaves):
        u_r, u_c, u_v, v_r, v_c, v_v = [], [], [], [], [], []
        slot = 0
        for (r0, c0, u, vt) in leaves:
            r = u.shape[1]
            if r == 0:
                continue
            mm, kk = u.shape[0], vt.shape[1]
            ui, uj = np.mgrid[0:mm, 0:r]
            u_r.append((ui + r0).ravel())
            u_c.append((uj + slot).ravel())
            u_v.append(u.ravel())
            vi, vj = np.mgrid[0:r, 0:kk]
            v_r.append((vi + slot).ravel())
            v_c.append((vj + c0).ravel())
            v_v.append(vt.ravel())
            slot += r

        def csr(shape, ri, ci, vv):
            if not ri:
                return sp.csr_matrix(shape, dtype=np.complex128)
            return sp.csr_matrix((np.concatenate(vv), (np.concatenate(ri), np.concatenate(ci))),
                                 shape=shape, dtype=np.complex128)

        self.left = csr((m, slot), u_r, u_c, u_v)
        self.right = csr((slot, m), v_r, v_c, v_v)
        self.shape = (m, m)

    def matvec(self, x):  # plr.py:253-259
        return self.left @ (self.right @ x)

    def to_dense(self):
        return (self.left @ self.right).toarray()


def operator_from_case(meta, arrays):
    """Rebuild (pol, perm) from PTC1 arrays written by tools/make_cases.py."""
    m = int(meta["m"])
    nb = 2 * int(meta["nt"]) if "nt" in meta else int(meta["n_block_rows"])
    kernels = []
    if "dense" in arrays:
        kernels = [np.asarray(k) for k in arrays["dense"]]
    else:
        leaves = np.asarray(arrays["leaves"])
        fac = np.asarray(arrays["factors"])
        nk = int(np.asarray(arrays["entries"])[:, 2].max()) + 1
        per = [[] for _ in range(nk)]
        for (k, r0, c0, mm, kk, r, uo, vo) in leaves:
            u = fac[uo:uo + mm * r].reshape(mm, r)
            vt = fac[vo:vo + r * kk].reshape(r, kk)
            per[int(k)].append((int(r0), int(c0), u, vt))
        kernels = [SparsePair(m, lv) for lv in per]
    pol = BlockMatrix(nb, nb, m)
    for (i, j, k), (s, e) in zip(np.asarray(arrays["entries"]), np.asarray(arrays["coefs"])):
        pol.entries[(int(i), int(j))] = Block(None if k < 0 else kernels[int(k)], s, e)
    return pol, np.asarray(arrays["perm"], dtype=np.intp)


def sweep_permutation(L):  # trace_system.py:353-365
    nt = 2 * L - 2
    down, up = [], []
    for i in range(1, L):
        down += [2 * i - 2, nt + 2 * i - 2]
        up += [nt + 2 * i - 1, 2 * i - 1]
    return np.array(down + up, dtype=np.intp)


def split_dr(pol, perm):  # trace_system.py:499-524
    """Returns ((D_down, D_up), (R_upper, R_lower)) sharing the entries of pol."""
    if pol.n_block_rows != pol.n_block_cols or pol.n_block_rows % 2:
        raise ValueError("polarized matrix must be square with an even block count")
    nt = pol.n_block_rows // 2
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    dd, du, ru, rl = (BlockMatrix(nt, nt, pol.m) for _ in range(4))
    for (i, j), e in pol.entries.items():
        pos = inv[i]
        if pos < nt:
            (dd if j < nt else ru).entries[(pos, j % nt)] = e
        else:
            (rl if j < nt else du).entries[(pos - nt, j % nt)] = e
    return (dd, du), (ru, rl)


def solve_block_triangular(tri, rhs, kind):  # trace_system.py:527-548
    m, nb = tri.m, tri.n_block_rows
    if rhs.shape != (nb * m,):
        raise ValueError("rhs length does not match the block layout")
    order = range(nb) if kind == "lower" else range(nb - 1, -1, -1)
    rows = tri.rows()
    x = np.zeros(nb * m, dtype=np.complex128)
    for i in order:
        acc = -rhs[i * m:(i + 1) * m]
        for j, e in rows[i]:
            if j == i:
                if not (e.kernel is None and e.eye == -1):
                    raise ValueError(f"diagonal block {i} is not exactly -I")
            else:
                acc = acc + e.apply(x[j * m:(j + 1) * m])
        x[i * m:(i + 1) * m] = acc
    return x


def gs_sweep(d, r, perm, rhs, u_in):  # solver.py:203-220
    d_down, d_up = d
    r_upper, r_lower = r
    nt, m = d_down.n_block_rows, d_down.m
    rp = np.asarray(rhs).reshape(2 * nt, m)[perm]
    u_in = np.asarray(u_in)
    if u_in.shape[0] != 2 * nt * m:
        raise ValueError(f"polarized vector has length {u_in.shape[0]}, expected {2 * nt * m}")
    g_down = rp[:nt].ravel() - r_upper.matvec(u_in[nt * m:])
    g_up = rp[nt:].ravel() - r_lower.matvec(u_in[:nt * m])
    return np.concatenate([solve_block_triangular(d_down, g_down, "lower"),
                           solve_block_triangular(d_up, g_up, "upper")])


def preconditioner_apply(n_it, d, r, perm, residual):  # solver.py:223-228
    u = np.zeros_like(np.asarray(residual, dtype=np.complex128))
    for _ in range(n_it):
        u = gs_sweep(d, r, perm, residual, u)
    return u


class OracleReport:
    def __init__(self):
        self.iterations = 0
        self.residual_history = []
        self.converged = False
        self.flag = "converged"
        self.true_residual = None


def gmres_solve(apply_A, apply_Minv, b, rel_tol=1e-7, max_iter=100):  # solver.py:231-295
    """MGS Arnoldi, lstsq per iteration, no restart; same flags as the reference."""
    b = np.asarray(b, dtype=np.complex128)
    rep = OracleReport()
    mb = apply_Minv(b)
    beta = np.linalg.norm(mb)
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128)
    if beta == 0.0:
        rep.converged, rep.true_residual = True, 0.0
        return x, rep
    V = np.zeros((n, max_iter + 1), dtype=np.complex128)
    V[:, 0] = mb / beta
    H = np.zeros((max_iter + 1, max_iter), dtype=np.complex128)
    e1 = np.zeros(max_iter + 1, dtype=np.complex128)
    e1[0] = beta
    y = np.zeros(0)
    k = 0
    for j in range(max_iter):
        w = apply_Minv(apply_A(V[:, j]))
        if not np.all(np.isfinite(w)):
            raise RuntimeError(f"non-finite values in preconditioned matvec at iteration {j + 1}")
        for i in range(j + 1):
            H[i, j] = np.vdot(V[:, i], w)
            w = w - H[i, j] * V[:, i]
        hn = np.linalg.norm(w)
        H[j + 1, j] = hn
        k = j + 1
        breakdown = hn <= 1e-14 * beta
        if not breakdown:
            V[:, j + 1] = w / hn
        y = np.linalg.lstsq(H[:k + 1, :k], e1[:k + 1], rcond=None)[0]
        rel = np.linalg.norm(e1[:k + 1] - H[:k + 1, :k] @ y) / beta
        rep.residual_history.append(float(rel))
        rep.iterations = k
        if breakdown:
            rep.converged, rep.flag = True, "breakdown"
            break
        if rel <= rel_tol:
            rep.converged = True
            break
        if len(rep.residual_history) > STAGNATION_WINDOW:
            old = rep.residual_history[-STAGNATION_WINDOW - 1]
            if old > 0 and 1.0 - rel / old < STAGNATION_IMPROVEMENT:
                rep.flag = "stagnation"
                break
    else:
        rep.flag = "maxiter"
    x = V[:, :k] @ y
    true_res = np.linalg.norm(b - apply_A(x))
    scale = np.linalg.norm(b)
    rep.true_residual = float(true_res / scale) if scale > 0 else float(true_res)
    return x, rep
