"""Pin c4 (1600x800, L=32, PLR) to the reference (test infrastructure).

The reference's own offline stage at c4 takes hours here, so the c4 operator
comes from the restated offline stage (paper_1410_5910_b200/offline).  This
script ties it to the REFERENCE (``/root/reference/pkg/src``, only present in
the build container) in two ways and records the results in
``tests/golden/c4_ref.ptc``:

1. per-layer pin: for a few layers, the reference's own layer pipeline --
   ``extend_slowness`` (partition.py:116-122), ``assemble_local``
   (grid.py:282-289), ``factorize(method="sparse")``,
   ``extract_interface_greens`` (local_solver.py:112-135) and ``compress``
   (plr.py:225-235) with ``CompressionConfig.resolve`` -- and the leaf
   structure (offsets, sizes, ranks) and per-leaf factor norms of every
   kernel of those layers (checked by ``offline.build.build_case``);
2. the reference's own online solve on that operator: the kernels wrapped as
   the reference's ``PLRSparseForm`` (plr.py:238-265), ``BlockEntry`` /
   ``BlockInterfaceMatrix`` (trace_system.py:145-226), ``split_DR``,
   ``preconditioner_apply`` and ``gmres_solve`` (solver.py:203-295): its
   iterations, residual history and traces, and probe applies (A and M on
   the seeded vector of tools/make_cases.py, every 16th entry).

    python tools/make_c4_ref.py /tmp/cases/c4.ptc [--layers 1 16 32]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
sys.path.insert(0, str(ROOT))

import make_cases as MC  # noqa: E402  (imports the reference package)
from helmsweep.grid import assemble_local  # noqa: E402
from helmsweep.local_solver import extract_interface_greens, factorize  # noqa: E402
from helmsweep.partition import extend_slowness  # noqa: E402
from helmsweep.plr import PLRSparseForm  # noqa: E402
from helmsweep.solver import gmres_solve, split_DR  # noqa: E402
from helmsweep.trace_system import BlockInterfaceMatrix  # noqa: E402

from paper_1410_5910_b200.cache import write_case  # noqa: E402
from paper_1410_5910_b200.operator import load_case_arrays  # noqa: E402

PROBE_STEP = 16


def layer_pin(ell, meta):
    """The reference's kernels of layer ell: {kernel index: [(r0, c0, m, k, rank, |U|)]}."""
    cfg = MC.config("c4")
    grid, L = cfg["grid"], cfg["L"]
    part = MC.make_partition(grid.nz, L)
    model = MC.model_from_c(grid, cfg["c"])
    n_layer = part.thickness(ell)
    t0 = time.perf_counter()
    op = assemble_local(grid, extend_slowness(model, part, ell, grid.n_pml), n_layer, float(cfg["omega"]))
    fact = factorize(op, method="sparse", label=f"layer {ell}")
    greens = extract_interface_greens(fact, n_layer, grid.n_pml, grid.h)
    eps, r_max = cfg["compression"].resolve(L, grid.nx_ext)
    out = {}
    for idx, key in enumerate(meta["kernel_keys"]):
        if int(key[0]) != ell or key[1] == "E":
            continue
        plr = MC_compress(greens.blocks[(int(key[1]), int(key[2]))], r_max, eps)
        out[idx] = [(r0, c0, lf.u.shape[0], lf.vt.shape[1], lf.rank, float(np.linalg.norm(lf.u)))
                    for (r0, c0, lf, _d) in plr.leaves() if lf.rank > 0]
    print(f"[c4] reference layer {ell}: {len(out)} kernels in {time.perf_counter() - t0:.0f} s", flush=True)
    return out


def MC_compress(block, r_max, eps):
    from helmsweep.plr import compress
    return compress(block, r_max=r_max, epsilon=eps)


def reference_operator(meta, arr):
    """Our c4 kernels as the reference's PLRSparseForm objects, in its
    BlockInterfaceMatrix (kernels shared by reference, as assemble_polarized does)."""
    m = int(meta["m"])
    nb = 2 * int(meta["nt"])
    leaves = np.asarray(arr["leaves"])
    fac = np.asarray(arr["factors"])
    nk = int(leaves[:, 0].max()) + 1
    per = [[] for _ in range(nk)]
    for row in leaves:
        per[int(row[0])].append(row)
    kernels = []
    for lv in per:
        ur, uc, uv, vr, vc, vv = [], [], [], [], [], []
        slot = 0
        for (_k, r0, c0, mm, kk, r, uo, vo) in lv:
            if r == 0:
                continue
            ui, uj = np.mgrid[0:mm, 0:r]
            ur.append((ui + r0).ravel())
            uc.append((uj + slot).ravel())
            uv.append(fac[uo:uo + mm * r])
            vi, vj = np.mgrid[0:r, 0:kk]
            vr.append((vi + slot).ravel())
            vc.append((vj + c0).ravel())
            vv.append(fac[vo:vo + r * kk])
            slot += int(r)
        left = sp.csr_matrix((np.concatenate(uv), (np.concatenate(ur), np.concatenate(uc))),
                             shape=(m, slot), dtype=np.complex128)
        right = sp.csr_matrix((np.concatenate(vv), (np.concatenate(vr), np.concatenate(vc))),
                              shape=(slot, m), dtype=np.complex128)
        kernels.append(PLRSparseForm(left, right, (m, m)))
    pol = BlockInterfaceMatrix(nb, nb, m)
    for (i, j, k), (s, e) in zip(np.asarray(arr["entries"]), np.asarray(arr["coefs"])):
        pol.add(int(i), int(j), None if k < 0 else kernels[int(k)], scale=s, eye=e)
    return pol, np.asarray(arr["perm"], dtype=np.intp)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--layers", type=int, nargs="+", default=[1, 16, 32])
    args = ap.parse_args()
    meta, arr = load_case_arrays(args.case)
    # 1. per-layer pin against the reference's own layer pipeline
    pin_k, pin_leaves = [], []
    worst = 0.0
    ours = np.asarray(arr["leaves"])
    fac = np.asarray(arr["factors"])
    for ell in args.layers:
        for idx, ref in layer_pin(ell, meta).items():
            mine = [row for row in ours if int(row[0]) == idx and row[5] > 0]
            if [tuple(int(v) for v in row[1:6]) for row in mine] != [r[:5] for r in ref]:
                raise SystemExit(f"kernel {idx}: leaf structure differs from the reference's")
            for row, r in zip(mine, ref):
                nrm = np.linalg.norm(fac[row[6]:row[6] + row[3] * row[5]])
                worst = max(worst, abs(nrm - r[5]) / max(r[5], 1e-300))
                pin_k.append(idx)
                pin_leaves.append(list(r[:5]) + [r[5]])
    print(f"[c4] layers {args.layers}: leaf structure identical, factor norms within {worst:.2e}",
          flush=True)
    # 2. the reference's online solve on this operator
    pol, perm = reference_operator(meta, arr)
    d, r = split_DR(pol, perm)
    from helmsweep.solver import GmresConfig, PreconditionerConfig, preconditioner_apply
    M = lambda v: preconditioner_apply(PreconditionerConfig(n_it=2), d, r, perm, v)  # noqa: E731
    N = 2 * int(meta["nt"]) * int(meta["m"])
    rng = np.random.default_rng(1234)
    px = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    t0 = time.perf_counter()
    ax = pol.matvec(px)
    mx = M(px)
    t_apply = time.perf_counter() - t0
    b = np.asarray(arr["rhs"][0])
    t0 = time.perf_counter()
    x, rep = gmres_solve(pol.matvec, M, b, GmresConfig(rel_tol=float(meta["gmres_tol"])))
    t_solve = time.perf_counter() - t0
    nt, m = int(meta["nt"]), int(meta["m"])
    traces = x[:nt * m] + x[nt * m:]
    print(f"[c4] reference gmres_solve: {rep.iterations} iterations, flag {rep.flag}, "
          f"{t_solve:.0f} s", flush=True)
    golden = {
        "rhs": b[None, :], "ref_traces": traces[None, :],
        "ref_hist": np.asarray(rep.residual_history)[None, :], "ref_index": np.asarray([0]),
        "probe_Ax_sub": ax[::PROBE_STEP], "probe_Mx_sub": mx[::PROBE_STEP],
        "probe_Ax_norm": np.asarray([np.linalg.norm(ax)]), "probe_Mx_norm": np.asarray([np.linalg.norm(mx)]),
        "ck_pin_kernel": np.asarray(pin_k, dtype=np.int64),
        "ck_pin_leaves": np.asarray(pin_leaves, dtype=np.float64),
    }
    gmeta = {"name": "c4", "note": meta["note"], "nx": meta["nx"], "nz": meta["nz"],
             "n_pml": meta["n_pml"], "L": meta["L"], "m": m, "nt": nt, "N": N,
             "gmres_tol": meta["gmres_tol"], "gmres_max_iter": 100, "n_it": 2,
             "kernel_format": "plr", "kernel_bytes": meta["kernel_bytes"],
             "probe_step": PROBE_STEP, "pinned_layers": args.layers,
             "pin_factor_norm_rel_err": worst,
             "solves": [{"label": "rhs[0]", "iterations": rep.iterations, "flag": rep.flag,
                         "converged": bool(rep.converged), "true_residual": rep.true_residual,
                         "stage_seconds": {"gmres": t_solve}}],
             "probe_apply_seconds": {"A+M": t_apply},
             "generator": "tools/make_c4_ref.py (reference helmsweep layer pipeline and online "
                          "solve on the restated c4 operator)"}
    out = ROOT / "tests" / "golden" / "c4_ref.ptc"
    write_case(out, gmeta, golden)
    print(f"[c4] wrote {out} ({out.stat().st_size / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    main()
