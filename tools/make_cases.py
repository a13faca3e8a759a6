"""Build PTC1 operator caches and golden results by running the REFERENCE here.

This script is test/bench infrastructure, not product code.  It imports the
reference package (``/root/reference/pkg/src``, only present in the build
container), builds each BASELINE configuration through the reference's own
public API -- ``ComplexGrid2D``, ``SquaredSlownessModel.from_interior``,
``make_partition``, ``offline_assemble`` (``solver.py:132-193``) and
``solve_helmholtz`` (``solver.py:308-435``) -- and records:

* the operator exactly as ``offline_assemble`` produced it: the entry table
  of ``state.pol`` (``trace_system.py:183-226``), ``state.perm``, and every
  distinct kernel (dense ``InterfaceGreens`` blocks, or the PLR leaves
  recovered from the reference's own ``PLRSparseForm`` factors,
  ``plr.py:239-297``);
* the polarized right-hand side the pipeline hands to GMRES
  (``polarized_rhs``, ``trace_system.py:475-484``);
* the reference's own results: GMRES solution, iterations, residual history,
  flag, true residual, traces and the reconstructed volume field;
* probe applies on seeded vectors: ``pol.matvec``, ``preconditioner_apply``
  (n_it 1 and 2) and one ``gs_sweep`` with a nonzero iterate.

Media follow SURVEY.md §8(d) (seeded synthetic stand-ins; no public dataset).

Usage::

    python tools/make_cases.py fixtures            # small cases -> tests/golden/
    python tools/make_cases.py c1 c3r c2 c5        # -> cases/*.ptc (git-ignored)
    python tools/make_cases.py c3                  # ~30 min, ~11 GB RSS
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, REF_SRC)

from helmsweep.grid import ComplexGrid2D, SquaredSlownessModel  # noqa: E402
from helmsweep.partition import make_partition  # noqa: E402
from helmsweep.solver import (  # noqa: E402
    CompressionConfig,
    GmresConfig,
    PreconditionerConfig,
    gs_sweep,
    offline_assemble,
    preconditioner_apply,
    solve_helmholtz,
)
from helmsweep.trace_system import polarized_rhs  # noqa: E402

from paper_1410_5910_b200.cache import write_case  # noqa: E402


# ----------------------------------------------------------------------------
# media and sources


def interior_xz(grid):
    x = grid.x_coords()[grid.interior_x_slice()]
    z = grid.z_coords()[grid.interior_z_slice()]
    return np.meshgrid(x, z)


def model_from_c(grid, c):
    return SquaredSlownessModel.from_interior(1.0 / c**2, grid.n_pml)


def medium_homogeneous(grid, c0=1.0):
    return np.full((grid.nz, grid.nx), float(c0))


def medium_gradient(grid):
    X, Z = interior_xz(grid)
    return 1.0 + 0.1 * X + 0.1 * Z


def medium_bumps(grid, seed=2, count=12):
    X, Z = interior_xz(grid)
    rng = np.random.default_rng(seed)
    c = np.full_like(X, 1.5)
    for _ in range(count):
        xk = rng.uniform(0.0, 1.0, size=2)
        ak = rng.uniform(-0.5, 1.5)
        wk = rng.uniform(0.05, 0.2)
        c = c + ak * np.exp(-((X - xk[0]) ** 2 + (Z - xk[1]) ** 2) / (2 * wk**2))
    return np.clip(c, 1.5, 4.5)


def medium_layered(grid, seed=3, n_layers=20, amp_h=3.0):
    X, Z = interior_xz(grid)
    rng = np.random.default_rng(seed)
    vel = rng.uniform(1.5, 5.5, size=n_layers)
    count = np.zeros(X.shape, dtype=np.int64)
    for k in range(1, n_layers):
        kappa = rng.uniform(1.0, 4.0)
        phi = rng.uniform(0.0, 2 * np.pi)
        zk = k * grid.Lz / n_layers + amp_h * grid.h * np.sin(2 * np.pi * kappa * X / grid.Lx + phi)
        count += (Z > zk).astype(np.int64)
    return vel[count]


def source_point(grid, fx, fz, amp=1.0):
    f = np.zeros((grid.nz_ext, grid.nx_ext), dtype=np.complex128)
    px = min(max(int(round(fx * (grid.nx + 1))), 1), grid.nx)
    qz = min(max(int(round(fz * (grid.nz + 1))), 1), grid.nz)
    f[grid.n_pml + qz - 1, grid.n_pml + px - 1] = amp / grid.h**2
    return f


def source_gaussian(grid, fx, fz, sigma):
    f = np.zeros((grid.nz_ext, grid.nx_ext), dtype=np.complex128)
    x = grid.x_coords()
    z = grid.z_coords()[grid.interior_z_slice()]
    X, Z = np.meshgrid(x, z)
    x0, z0 = fx * grid.Lx, fz * grid.Lz
    g = np.exp(-((X - x0) ** 2 + (Z - z0) ** 2) / (2 * sigma**2)) / (2 * np.pi * sigma**2)
    f[grid.interior_z_slice(), :] = g
    return f


def source_random(grid, seed):
    rng = np.random.default_rng(seed)
    f = np.zeros((grid.nz_ext, grid.nx_ext), dtype=np.complex128)
    shape = (grid.nz, grid.nx_ext)
    f[grid.interior_z_slice(), :] = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return f


# ----------------------------------------------------------------------------
# configurations


def _grid(nx, nz, n_pml):
    return ComplexGrid2D(nx=nx, nz=nz, h=1.0 / (nx + 1), n_pml=n_pml)


def config(name):
    """Return dict(grid, c, L, omega, sources, compression, tol, note)."""
    if name == "c1":
        g = _grid(200, 200, 20)
        c = medium_homogeneous(g)
        return dict(grid=g, c=c, L=4, omega=2 * np.pi * 20,
                    sources=[("gauss", source_gaussian(g, 0.5, 0.1, 2 * g.h))],
                    compression=None, tol=1e-9,
                    note="homogeneous c=1, 200^2+20 PML, omega=2pi*20, L=4, Gaussian source sigma=2h, dense")
    if name in ("c2", "c5"):
        g = _grid(400, 400, 30)
        c = medium_bumps(g)
        omega = 2 * np.pi * c.min() / (10 * g.h)
        if name == "c2":
            src = [("point", source_point(g, 0.5, 0.1))]
            note = "12 seeded Gaussian bumps (rng 2), 400^2+30 PML, 10 ppw, L=8, point source, dense"
        else:
            src = [(f"point{s}", source_point(g, (s + 0.5) / 64, 0.05)) for s in range(64)]
            note = "c2 medium and layering, 64 point sources at depth 0.05 (multi-RHS batch)"
        return dict(grid=g, c=c, L=8, omega=omega, sources=src, compression=None, tol=1e-9, note=note)
    if name == "c3":
        g = _grid(800, 800, 40)
        c = medium_layered(g)
        omega = 2 * np.pi * c.min() / (8 * g.h)
        return dict(grid=g, c=c, L=16, omega=omega,
                    sources=[("point", source_point(g, 0.5, 0.1))],
                    compression=CompressionConfig(epsilon=1e-9, r_max=32), tol=1e-9,
                    note="20 seeded layers (rng 3) with 3h undulation, 800^2+40 PML, 8 ppw, L=16, point source, PLR eps 1e-9 r_max 32")
    if name == "c3r":
        g = _grid(160, 160, 16)
        c = medium_layered(g)
        omega = 2 * np.pi * c.min() / (8 * g.h)
        return dict(grid=g, c=c, L=4, omega=omega,
                    sources=[("point", source_point(g, 0.5, 0.1))],
                    compression=CompressionConfig(epsilon=1e-9, r_max=32), tol=1e-9,
                    note="reduced c3: layered medium 160^2+16 PML, 8 ppw, L=4, PLR eps 1e-9 r_max 32")
    # ---- small fixtures (tests/golden) ----
    if name == "fx_tiny":
        g = _grid(8, 9, 3)
        return dict(grid=g, c=medium_gradient(g), L=3, omega=4.0,
                    sources=[("rand", source_random(g, 7))], compression=None, tol=1e-10,
                    note="reference test_solver.py tiny geometry: 8x9, L=3, n_pml=3, omega=4, gradient")
    if name == "fx_l2":
        g = _grid(12, 12, 4)
        return dict(grid=g, c=medium_gradient(g), L=2, omega=6.0,
                    sources=[("point", source_point(g, 0.4, 0.3))], compression=None, tol=1e-10,
                    note="L=2 edge case (no kernel-bearing sweep steps)")
    if name == "fx_uneven":
        g = _grid(10, 19, 4)
        return dict(grid=g, c=medium_gradient(g), L=4, omega=7.0,
                    sources=[("point", source_point(g, 0.5, 0.7))], compression=None, tol=1e-10,
                    note="uneven layers 5,5,5,4 (remainder to the front), L=4")
    if name == "fx_plr":
        g = _grid(40, 40, 10)
        return dict(grid=g, c=medium_gradient(g), L=4, omega=9.0,
                    sources=[("point", source_point(g, 0.5, 0.25))],
                    compression=CompressionConfig(epsilon=1e-9, r_max=4), tol=1e-10,
                    note="PLR with real quadtree splits: m=60, r_max=4 (min leaf 8), L=4")
    if name == "fx_plr_odd":
        g = _grid(37, 30, 8)
        return dict(grid=g, c=medium_layered(g, seed=5, n_layers=5, amp_h=1.0), L=3, omega=11.0,
                    sources=[("point", source_point(g, 0.3, 0.5))],
                    compression=CompressionConfig(epsilon=1e-6, r_max=3), tol=1e-10,
                    note="PLR with odd m=53 (floor-first splits), eps 1e-6 (rank-deficient leaves), L=3")
    raise KeyError(name)


# ----------------------------------------------------------------------------
# operator capture


def _leaves_from_sparse_form(sf):
    """Recover quadtree leaves from the reference's PLRSparseForm (plr.py:268-297).

    Slots are assigned leaf by leaf in preorder; a leaf occupies a run of
    consecutive slots sharing one row range (in ``left``) and one column
    range (in ``right``).  Explicit zeros are stored, so the ranges are exact.
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
        assert left.indptr[s + 1] - left.indptr[s] == r1 - r0
        assert right.indptr[s + 1] - right.indptr[s] == c1 - c0
        u = sf.left[r0:r1, s:e].toarray()
        vt = sf.right[s:e, c0:c1].toarray()
        leaves.append((r0, c0, u, vt))
        s = e
    return leaves


def capture_operator(state):
    pol = state.pol
    m = pol.m
    items = sorted(pol.entries.items())
    kid = {}
    kernels = []
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
    arrays = {"entries": entries, "coefs": coefs, "perm": np.asarray(state.perm, dtype=np.int64)}
    if all(isinstance(k, np.ndarray) for k in kernels):
        arrays["dense"] = np.stack([np.asarray(k, dtype=np.complex128) for k in kernels])
        fmt = "dense"
        kbytes = [16 * m * m] * len(kernels)
    else:
        fmt = "plr"
        leaf_rows, chunks, kl = [], [], []
        off = 0
        kbytes = []
        for k_id, sf in enumerate(kernels):
            leaves = _leaves_from_sparse_form(sf)
            kl.append((len(leaf_rows), len(leaves)))
            nb = 0
            for (r0, c0, u, vt) in leaves:
                ml, r = u.shape
                kk = vt.shape[1]
                leaf_rows.append((k_id, r0, c0, ml, kk, r, off, off + ml * r))
                chunks.append(np.ascontiguousarray(u).ravel())
                chunks.append(np.ascontiguousarray(vt).ravel())
                off += ml * r + r * kk
                nb += 16 * r * (ml + kk)
            assert nb == 16 * sf.stored_entries(), (nb, sf.stored_entries())
            kbytes.append(nb)
            # the recovered leaves must reproduce the reference factor product
            dense = np.zeros((m, m), dtype=np.complex128)
            for (r0, c0, u, vt) in leaves:
                dense[r0:r0 + u.shape[0], c0:c0 + vt.shape[1]] += u @ vt
            ref = sf.to_dense()
            scale = max(np.abs(ref).max(), 1e-300)
            assert np.abs(dense - ref).max() <= 1e-12 * scale
        arrays["leaves"] = np.asarray(leaf_rows, dtype=np.int64).reshape(-1, 8)
        arrays["kernel_leaves"] = np.asarray(kl, dtype=np.int64).reshape(-1, 2)
        arrays["factors"] = np.concatenate(chunks) if chunks else np.zeros(0, np.complex128)
    return fmt, arrays, kbytes


# ----------------------------------------------------------------------------


def build(name, out_dir, operator_from=None, state_cache={}):
    cfg = config(name)
    grid, L = cfg["grid"], cfg["L"]
    part = make_partition(grid.nz, L)
    model = model_from_c(grid, cfg["c"])
    omega = float(cfg["omega"])
    op_key = "c2" if name == "c5" else name
    t0 = time.perf_counter()
    if op_key in state_cache:
        state = state_cache[op_key]
        offline_s = None
    else:
        state = offline_assemble(grid, model, part, omega, factor_method="sparse",
                                 compression=cfg["compression"])
        offline_s = time.perf_counter() - t0
        state_cache[op_key] = state
    print(f"[{name}] offline {offline_s}s stages={state.stage_seconds}", flush=True)

    m = state.block_size
    nt = state.n_traces
    N = 2 * nt * m
    meta = {
        "name": name, "note": cfg["note"], "nx": grid.nx, "nz": grid.nz, "n_pml": grid.n_pml,
        "h": grid.h, "L": L, "n_c": list(part.n_c), "omega": omega, "m": m, "nt": nt, "N": N,
        "c_min": float(cfg["c"].min()), "c_max": float(cfg["c"].max()),
        "variant": state.variant, "gmres_tol": cfg["tol"], "gmres_max_iter": 100, "n_it": 2,
        "offline_seconds": offline_s,
        "offline_stage_seconds": {k: float(v) for k, v in state.stage_seconds.items()},
        "compression": None if cfg["compression"] is None else
        {"epsilon": cfg["compression"].epsilon, "r_max": cfg["compression"].r_max},
        "generator": "tools/make_cases.py (reference helmsweep, numpy %s)" % np.__version__,
    }
    arrays = {}
    if name == "c5":
        meta["operator_case"] = "c2"
    else:
        fmt, op_arrays, kbytes = capture_operator(state)
        meta["kernel_format"] = fmt
        meta["n_kernels"] = len(kbytes)
        meta["kernel_bytes"] = int(sum(kbytes))
        arrays.update(op_arrays)
        arrays["kernel_bytes"] = np.asarray(kbytes, dtype=np.int64)

    # probe applies on seeded vectors (per-apply parity targets)
    rng = np.random.default_rng(1234)
    px = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    pu = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    arrays["probe_x"] = px
    arrays["probe_u"] = pu
    t = time.perf_counter()
    arrays["probe_Ax"] = state.pol.matvec(px)
    ta = time.perf_counter() - t
    t = time.perf_counter()
    arrays["probe_Mx"] = preconditioner_apply(PreconditionerConfig(n_it=2), state.d, state.r, state.perm, px)
    tm = time.perf_counter() - t
    arrays["probe_M1x"] = preconditioner_apply(PreconditionerConfig(n_it=1), state.d, state.r, state.perm, px)
    arrays["probe_sweep"] = gs_sweep(state.d, state.r, state.perm, px, pu)
    meta["probe_apply_seconds"] = {"A": ta, "M": tm}

    # reference solves
    gm = GmresConfig(rel_tol=cfg["tol"])
    rhs_list, x_list, tr_list, hist_list, recs = [], [], [], [], []
    u0 = None
    for s, (label, f) in enumerate(cfg["sources"]):
        rep = solve_helmholtz(model, grid, part, f, state=state, gmres=gm)
        # the polarized rhs the pipeline handed to GMRES, and its solution x
        from helmsweep.local_solver import newton_trace
        from helmsweep.partition import restrict_source
        newtons = [newton_trace(state.facts[ell - 1], restrict_source(f, part, ell, grid.n_pml),
                                part.thickness(ell), grid.n_pml) for ell in range(1, L + 1)]
        rhs = polarized_rhs(newtons, part, state.variant)
        from helmsweep.solver import gmres_solve
        x, inner = gmres_solve(state.pol.matvec,
                               lambda r: preconditioner_apply(PreconditionerConfig(), state.d, state.r, state.perm, r),
                               rhs, gm)
        assert inner.iterations == rep.iterations
        tr = rep.traces
        assert np.abs((x[:nt * m] + x[nt * m:]) - tr).max() <= 1e-12 * max(np.abs(tr).max(), 1e-300)
        rhs_list.append(rhs)
        x_list.append(x)
        tr_list.append(tr)
        hist_list.append(list(rep.residual_history))
        recs.append({"label": label, "iterations": rep.iterations, "flag": rep.flag,
                     "converged": bool(rep.converged), "true_residual": rep.true_residual,
                     "stage_seconds": {k: float(v) for k, v in rep.stage_seconds.items()}})
        if s == 0:
            u0 = rep.u
        print(f"[{name}] {label}: it={rep.iterations} flag={rep.flag} "
              f"gmres={rep.stage_seconds.get('gmres')}", flush=True)
    hmax = max((len(h) for h in hist_list), default=0)
    hist = np.full((len(hist_list), max(hmax, 1)), np.nan)
    for s, h in enumerate(hist_list):
        hist[s, :len(h)] = h
    arrays["rhs"] = np.stack(rhs_list)
    arrays["ref_x"] = np.stack(x_list)
    arrays["ref_traces"] = np.stack(tr_list)
    arrays["ref_hist"] = hist
    if u0 is not None and name != "c5":
        arrays["ref_u"] = u0
    meta["solves"] = recs
    out = Path(out_dir) / f"{name}.ptc"
    write_case(out, meta, arrays)
    print(f"[{name}] wrote {out} ({out.stat().st_size / 1e6:.1f} MB) in {time.perf_counter() - t0:.1f}s",
          flush=True)
    return out


FIXTURES = ["fx_tiny", "fx_l2", "fx_uneven", "fx_plr", "fx_plr_odd"]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    names = []
    for n in args.names:
        names += FIXTURES if n == "fixtures" else [n]
    for n in names:
        out = args.out or (ROOT / "tests" / "golden" if n.startswith("fx_") else ROOT / "cases")
        Path(out).mkdir(parents=True, exist_ok=True)
        build(n, out)


if __name__ == "__main__":
    main()
