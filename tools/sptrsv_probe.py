"""Feasibility probe (profiling aid): GPU sparse triangular solves on the
SuperLU factors of one c3 layer (torch -> cuSPARSE SpSV), timed.

    python tools/sptrsv_probe.py [case] [layer]
"""
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.offline.configs import config  # noqa: E402
from paper_1410_5910_b200.offline.layers import Layer, edge_extend, equal_partition  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = config(name)
g = cfg.geo
n_c = equal_partition(g.nz, cfg.L)
m_ext = edge_extend(1.0 / cfg.c**2, g.n_pml)
lo = g.n_pml + n_c[ell - 1]
n_layer = int(n_c[ell] - n_c[ell - 1])
t0 = time.perf_counter()
lay = Layer(g.nx, n_layer, g.h, g.n_pml, float(cfg.omega), edge_extend(m_ext[lo:lo + n_layer, :], g.n_pml, axis=0))
print(f"factor {time.perf_counter() - t0:.2f}s dim {lay.dim}", flush=True)
L, U = lay.lu.L.tocsr(), lay.lu.U.tocsr()
print("nnz L", L.nnz, "U", U.nnz, flush=True)
pr, pc = lay.lu.perm_r, lay.lu.perm_c
rng = np.random.default_rng(0)
b = rng.standard_normal(lay.dim) + 1j * rng.standard_normal(lay.dim)
x_ref = lay.lu.solve(b)
# Pr A Pc = L U  ->  x = Pc U^-1 L^-1 Pr b
y = np.empty_like(b)
y[pr] = b
import scipy.sparse.linalg as spla
w = spla.spsolve_triangular(L, y, lower=True)
z = spla.spsolve_triangular(U, w, lower=False)
x = np.empty_like(b)
x[pc] = z
print("host perm check", np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref), flush=True)
# levels (row dependency depth) of L and U
def levels(M, lower):
    M = M.tocsr()
    n = M.shape[0]
    lv = np.zeros(n, dtype=np.int64)
    order = range(n) if lower else range(n - 1, -1, -1)
    ip, ix = M.indptr, M.indices
    for i in order:
        cols = ix[ip[i]:ip[i + 1]]
        cols = cols[cols < i] if lower else cols[cols > i]
        lv[i] = 1 + (lv[cols].max() if len(cols) else 0)
    return lv.max()
print("levels L", levels(L, True), "U", levels(U, False), flush=True)
dev = "cuda"
def to_t(M):
    M = M.tocsr()
    return torch.sparse_csr_tensor(torch.from_numpy(M.indptr.astype(np.int64)), torch.from_numpy(M.indices.astype(np.int64)),
                                   torch.from_numpy(M.data.astype(np.complex128)), size=M.shape).to(dev)
Lt, Ut = to_t(L), to_t(U)
yt = torch.from_numpy(y).to(dev).reshape(-1, 1)
for k in (1, 3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        wt = torch.linalg.solve_triangular(Lt, yt, upper=False, unitriangular=False)
        zt = torch.linalg.solve_triangular(Ut, wt, upper=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k
    print(f"torch sparse solve_triangular L+U: {dt * 1e3:.2f} ms", flush=True)
xt = np.empty_like(b)
xt[pc] = zt.cpu().numpy().ravel()
print("gpu err", np.linalg.norm(xt - x_ref) / np.linalg.norm(x_ref))
