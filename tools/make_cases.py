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
# configurations: one definition, shared with the GPU-box builder


def config(name):
    """The package's CaseConfig mapped onto the reference's own objects."""
    from paper_1410_5910_b200.offline.configs import config as pkg_config
    c = pkg_config(name)
    g = ComplexGrid2D(nx=c.geo.nx, nz=c.geo.nz, h=c.geo.h, n_pml=c.geo.n_pml)
    comp = None
    if c.compression is not None:
        comp = CompressionConfig(epsilon=c.compression[0], r_max=c.compression[1])
    return dict(grid=g, c=c.c, L=c.L, omega=c.omega, sources=c.sources, compression=comp,
                tol=c.tol, note=c.note, variant=c.variant)


def model_from_c(grid, c):
    return SquaredSlownessModel.from_interior(1.0 / c**2, grid.n_pml)


# ----------------------------------------------------------------------------
# operator capture


def capture_operator(state):
    from paper_1410_5910_b200.capture import capture_operator as cap
    meta, arrays = cap(state.pol, state.perm)
    return meta["kernel_format"], arrays, list(arrays["kernel_bytes"])


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
        state = offline_assemble(grid, model, part, omega, variant=cfg["variant"],
                                 factor_method="sparse", compression=cfg["compression"])
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
    pc = PreconditionerConfig(variant=cfg["variant"])
    rhs_list, x_list, tr_list, hist_list, recs = [], [], [], [], []
    u0 = None
    for s, (label, f) in enumerate(cfg["sources"]):
        rep = solve_helmholtz(model, grid, part, f, state=state, precond=pc, gmres=gm)
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


from paper_1410_5910_b200.offline.configs import FIXTURES  # noqa: E402
LITE_SUBSET = {"c5": list(range(0, 64, 9))}


def write_lite(name, full_dir=ROOT / "cases", out_dir=ROOT / "tests" / "golden"):
    """tests/golden/<name>_ref.ptc: the reference's results and operator
    checksums for a large case, without the kernels (which exceed what can be
    shipped to the GPU box; the box rebuilds them with
    paper_1410_5910_b200.offline.build and verifies them against these
    checksums)."""
    from paper_1410_5910_b200.cache import read_case
    from paper_1410_5910_b200.offline.build import operator_checksums
    from paper_1410_5910_b200.operator import load_case_arrays
    meta, arr = load_case_arrays(Path(full_dir) / f"{name}.ptc")
    ck = operator_checksums(meta, arr)
    idx = LITE_SUBSET.get(name, list(range(arr["rhs"].shape[0])))
    lite = dict(ck)
    lite["ref_index"] = np.asarray(idx, dtype=np.int64)
    for k in ("rhs", "ref_x", "ref_traces", "ref_hist"):
        lite[k] = np.asarray(arr[k])[idx]
    for k in ("probe_x", "probe_u", "probe_Ax", "probe_Mx", "probe_M1x", "probe_sweep"):
        lite[k] = np.asarray(arr[k])
    lmeta = {k: meta[k] for k in ("name", "note", "nx", "nz", "n_pml", "h", "L", "n_c", "omega",
                                  "m", "nt", "N", "c_min", "c_max", "gmres_tol", "gmres_max_iter",
                                  "n_it", "offline_seconds", "offline_stage_seconds",
                                  "probe_apply_seconds", "generator") if k in meta}
    lmeta["solves"] = [meta["solves"][i] for i in idx]
    lmeta["kernel_format"] = meta.get("kernel_format")
    lmeta["kernel_bytes"] = meta.get("kernel_bytes")
    out = Path(out_dir) / f"{name}_ref.ptc"
    write_case(out, lmeta, lite)
    print(f"[{name}] lite golden {out} ({out.stat().st_size / 1e6:.2f} MB)", flush=True)
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--out", default=None)
    ap.add_argument("--lite", action="store_true",
                    help="only write tests/golden/<name>_ref.ptc from an existing cases/<name>.ptc")
    args = ap.parse_args(argv)
    names = []
    for n in args.names:
        names += FIXTURES if n == "fixtures" else [n]
    for n in names:
        if args.lite:
            write_lite(n)
            continue
        out = args.out or (ROOT / "tests" / "golden" if n.startswith("fx_") else ROOT / "cases")
        Path(out).mkdir(parents=True, exist_ok=True)
        build(n, out)
        if not n.startswith("fx_"):
            write_lite(n)


if __name__ == "__main__":
    main()
