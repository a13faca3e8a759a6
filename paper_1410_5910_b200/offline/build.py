"""Build a PTC1 operator cache for a BASELINE configuration, layer-parallel.

    python -m paper_1410_5910_b200.offline.build c3 [--out DIR] [--workers N]

Layers are independent in the offline stage: each
worker process factorises one layer, extracts only the Green's blocks the
polarized system references, compresses them when the configuration asks
for PLR, and returns the Newton traces of the case's sources.  The parent
assembles the entry table and the right-hand sides, attaches the
reference's own results for the case (tests/golden/<case>_ref.ptc, written by
tools/make_cases.py from the reference package), checks the operator against
the reference's checksums, and writes ``<out>/<case>.ptc``.

This stays host code (the north star keeps the offline stage on the CPU); it
exists because the reference cannot run on the GPU box and its c2/c3 operator
caches exceed what can be shipped there.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

from ..cache import read_case, write_case
from .assemble import extrapolator, extrapolator_pairs, polarized_rhs, polarized_table
from .compress import leaf_table, plr_leaves
from .configs import config
from .layers import Layer, edge_extend, equal_partition, layer_operator

ROOT = Path(__file__).resolve().parents[2]
GOLDEN = ROOT / "tests" / "golden"
DEFAULT_OUT = Path(os.environ.get("PT_CASES", ROOT / "cases"))

__all__ = ["build_case", "ensure_case", "operator_checksums", "compare_checksums"]


def _layer_job(job):
    """Worker: factorise one layer, its Green's blocks (compressed), Newton traces."""
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(1)
    except Exception:  # pragma: no cover
        limiter = None
    t0 = time.perf_counter()
    lay = Layer(job["nx"], job["n_layer"], job["h"], job["n_pml"], job["omega"], job["m_tilde"])
    t1 = time.perf_counter()
    blocks = lay.greens(job["pairs"])
    t2 = time.perf_counter()
    out = {}
    for (j, k) in job["kernel_pairs"]:
        blk = blocks[(j, k)]
        out[(j, k)] = blk if job["compression"] is None else \
            plr_leaves(blk, r_max=job["compression"][1], eps=job["compression"][0])
    for d in job["extrapolators"]:  # dense, never compressed (trace_system.py:460-464)
        num, den = extrapolator_pairs(job["n_layer"], d)
        out[("E", d)] = extrapolator(blocks[num], blocks[den])
    t3 = time.perf_counter()
    newtons = [lay.newton(f) for f in job["f_local"]]
    if limiter is not None:
        limiter.unregister() if hasattr(limiter, "unregister") else None
    return job["ell"], out, newtons, {"factor": t1 - t0, "greens": t2 - t1, "compress": t3 - t2}


def _factor_job(job):
    """Worker (GPU offline): the layer operator factored in the device order."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass
    from .local import factor_layer
    t0 = time.perf_counter()
    op = layer_operator(job["nx"], job["n_layer"], job["h"], job["n_pml"], job["omega"], job["m_tilde"])
    fac = factor_layer(op, job["n_layer"] + 2 * job["n_pml"], job["nx"] + 2 * job["n_pml"], check=False)
    return job["ell"], fac, time.perf_counter() - t0


def _compress_job(args):
    """Worker (GPU offline): quadtree compression of one layer's blocks on the host."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass
    blocks, r_max, eps = args
    t0 = time.perf_counter()
    out = {p: plr_leaves(b, r_max=r_max, eps=eps) for p, b in blocks.items()}
    return out, time.perf_counter() - t0


def _layer_job_gpu(job, fac, device, compress_on="cuda"):
    """One layer on the GPU (offline.gpu): Green's blocks by multi-column
    sparse triangular solves, Newton traces by the same factors, and (with
    compress_on="cuda") PLR compression by batched SVDs; otherwise the dense
    blocks of the kernels that need compression are returned under
    "to_compress" for the host workers.  Same outputs as _layer_job."""
    import torch
    from .gpu import DeviceLayer, plr_leaves_gpu
    nze, nxe = job["n_layer"] + 2 * job["n_pml"], job["nx"] + 2 * job["n_pml"]
    t1 = time.perf_counter()
    lay = DeviceLayer(fac, nze, nxe, job["n_layer"], job["n_pml"], job["h"], device)
    blocks = lay.greens(job["pairs"])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out = {}
    if job["compression"] is None:
        for (j, k) in job["kernel_pairs"]:
            out[(j, k)] = blocks[(j, k)].cpu().numpy()
    elif compress_on == "cuda":
        leaves = plr_leaves_gpu([blocks[p] for p in job["kernel_pairs"]],
                                r_max=job["compression"][1], eps=job["compression"][0])
        for p, lv in zip(job["kernel_pairs"], leaves):
            out[p] = lv
    else:
        out["to_compress"] = {p: blocks[p].cpu().numpy() for p in job["kernel_pairs"]}
    for d in job["extrapolators"]:  # dense, never compressed (trace_system.py:460-464)
        num, den = extrapolator_pairs(job["n_layer"], d)
        out[("E", d)] = extrapolator(blocks[num].cpu().numpy(), blocks[den].cpu().numpy())
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    newtons = []
    n = job["n_layer"]
    q_in = lay.inv_in.argsort()
    for f in job["f_local"]:
        b = torch.from_numpy(np.ascontiguousarray(f, dtype=np.complex128).ravel()).to(lay.device)
        z = lay.solve_columns(b[q_in].unsqueeze(1))[:, 0]  # y = b[q_in]
        w = z[lay.q_out].reshape(nze, nxe)
        newtons.append({k: w[lay.row(k), :].cpu().numpy().copy() for k in (0, 1, n, n + 1)})
    del lay, blocks
    return job["ell"], out, newtons, {"greens": t2 - t1, "compress": t3 - t2}


# cases whose operator is another case's (same medium and layering)
OPERATOR_OF = {"c5": "c2"}


def build_operator(name, workers=None, sources=True, device=None, compress_on="host"):
    """``device`` (e.g. "cuda"): Green's extraction on the GPU (offline.gpu), the
    layer factorizations on the host workers, the PLR compression on the host
    workers as the blocks arrive (``compress_on="host"``) or by batched SVDs on
    the GPU (``"cuda"``: same leaves, but cuSOLVER's complex128 SVD of the large
    quadtree nodes is slower than the host workers)."""
    cfg = config(name)
    kernels_needed = name not in OPERATOR_OF
    g, L = cfg.geo, cfg.L
    n_c = equal_partition(g.nz, L)
    m_ext = edge_extend(1.0 / cfg.c**2, g.n_pml)
    variant = cfg.variant
    entries, coefs, keys, perm = polarized_table(n_c, g.h, variant)
    jobs = []
    for ell in range(1, L + 1):
        lo = g.n_pml + n_c[ell - 1]
        n_layer = int(n_c[ell] - n_c[ell - 1])
        rows = m_ext[lo:lo + n_layer, :]
        f_local = []
        if sources:
            for _, f in cfg.sources:
                fl = np.zeros((n_layer + 2 * g.n_pml, g.nx_ext), dtype=np.complex128)
                fl[g.n_pml:g.n_pml + n_layer, :] = f[lo:lo + n_layer, :]
                f_local.append(fl)
        kpairs = sorted({(j, k) for (l_, j, k) in keys if l_ == ell and j != "E"}) \
            if kernels_needed else []
        extr = sorted({k for (l_, j, k) in keys if l_ == ell and j == "E"}) if kernels_needed else []
        need = set(kpairs)
        for d in extr:
            need |= set(extrapolator_pairs(n_layer, d))
        jobs.append({"ell": ell, "nx": g.nx, "n_layer": n_layer, "h": g.h, "n_pml": g.n_pml,
                     "omega": float(cfg.omega), "m_tilde": edge_extend(rows, g.n_pml, axis=0),
                     "pairs": sorted(need), "kernel_pairs": kpairs, "extrapolators": extr,
                     "compression": cfg.compression, "f_local": f_local})
    workers = workers or min(L, os.cpu_count() or 1)
    t0 = time.perf_counter()
    if device is not None:
        # host workers factor the layers (in order), the GPU takes each layer
        # as its factors arrive, and the workers compress the layer's blocks
        # while the GPU extracts the next layer's
        results, pending = [], []

        def finish(r, compress):
            blocks = r[1].pop("to_compress", None)
            if blocks is not None:
                args = (blocks, cfg.compression[1], cfg.compression[0])
                pending.append((r, compress(args)))
            results.append(r)

        if workers > 1:
            import multiprocessing as mp
            ctx = mp.get_context("fork")
            with ctx.Pool(min(workers, L)) as pool:
                for ell, fac, t_fac in pool.imap(_factor_job, jobs, chunksize=1):
                    r = _layer_job_gpu(jobs[ell - 1], fac, device, compress_on)
                    r[3]["factor"] = t_fac
                    finish(r, lambda a: pool.apply_async(_compress_job, (a,)))
                for r, fut in pending:
                    leaves, t_c = fut.get()
                    r[1].update(leaves)
                    r[3]["compress"] += t_c
        else:
            for job in jobs:
                ell, fac, t_fac = _factor_job(job)
                r = _layer_job_gpu(job, fac, device, compress_on)
                r[3]["factor"] = t_fac
                finish(r, _compress_job)
            for r, (leaves, t_c) in pending:
                r[1].update(leaves)
                r[3]["compress"] += t_c
    elif workers > 1:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(min(workers, L)) as pool:
            results = pool.map(_layer_job, jobs, chunksize=1)
    else:
        results = [_layer_job(j) for j in jobs]
    wall = time.perf_counter() - t0
    per_layer = {ell: (out, newtons, st) for ell, out, newtons, st in results}
    arrays = {"entries": entries, "coefs": coefs, "perm": perm}
    meta = {"name": name, "note": cfg.note, "nx": g.nx, "nz": g.nz, "n_pml": g.n_pml, "h": g.h,
            "L": L, "n_c": [int(v) for v in n_c], "omega": float(cfg.omega), "m": g.nx_ext,
            "nt": 2 * L - 2, "N": 2 * (2 * L - 2) * g.nx_ext, "c_min": float(cfg.c.min()),
            "c_max": float(cfg.c.max()), "variant": variant, "gmres_tol": cfg.tol,
            "gmres_max_iter": 100, "n_it": 2, "n_kernels": len(keys),
            "kernel_keys": [list(k) for k in keys],
            "compression": None if cfg.compression is None else
            {"epsilon": cfg.compression[0], "r_max": cfg.compression[1]},
            "offline_seconds": wall, "offline_workers": workers,
            "offline_stage_seconds": {k: float(sum(v[2][k] for v in per_layer.values()))
                                      for k in ("factor", "greens", "compress")},
            "generator": "paper_1410_5910_b200.offline.build (restated reference offline" +
                         (f"; Green's extraction and compression on {device})" if device else ")")}
    if not kernels_needed:
        meta["operator_case"] = OPERATOR_OF[name]
        del arrays["entries"], arrays["coefs"], arrays["perm"]
    elif cfg.compression is None:
        kernels = [per_layer[ell][0][(j, k)] for (ell, j, k) in keys]  # (E, dir) for extrapolators
        meta["kernel_format"] = "dense"
        arrays["dense"] = np.stack(kernels)
        kb = np.full(len(keys), 16 * g.nx_ext**2, dtype=np.int64)
    else:
        kernels = [per_layer[ell][0][(j, k)] for (ell, j, k) in keys]
        meta["kernel_format"] = "plr"
        arrays["leaves"], arrays["factors"], kb = leaf_table(kernels)
    if kernels_needed:
        arrays["kernel_bytes"] = kb
        meta["kernel_bytes"] = int(kb.sum())
    if sources:
        rhs = [polarized_rhs([per_layer[ell][1][s] for ell in range(1, L + 1)], n_c, variant)
               for s in range(len(cfg.sources))]
        arrays["rhs"] = np.stack(rhs)
        meta["source_labels"] = [lbl for lbl, _ in cfg.sources]
    return meta, arrays


def operator_checksums(meta, arrays):
    """Per-kernel fingerprints that do not depend on SVD phase conventions."""
    out = {"entries": np.asarray(arrays["entries"]), "coefs": np.asarray(arrays["coefs"]),
           "perm": np.asarray(arrays["perm"])}
    if "dense" in arrays:
        d = np.asarray(arrays["dense"])
        out["ck_norm"] = np.sqrt((np.abs(d) ** 2).sum(axis=(1, 2)))
        out["ck_colsum"] = d.sum(axis=1)  # per kernel, per column: sensitive to every entry
    else:
        lv = np.asarray(arrays["leaves"])
        fac = np.asarray(arrays["factors"])
        out["ck_leaves"] = lv[:, :6].copy()
        nrm = np.empty(lv.shape[0])
        for i, (k, r0, c0, ml, kk, r, uo, vo) in enumerate(lv):
            nrm[i] = np.sqrt((np.abs(fac[uo:uo + ml * r]) ** 2).sum())
        out["ck_norm"] = nrm
    return out


def compare_pinned_layers(meta, arrays, ref, rtol=1e-9):
    """c4: the kernels of the layers the reference's own layer pipeline was run
    on (tools/make_c4_ref.py) -- leaf structure identical, factor norms within
    rtol.  Raises ValueError otherwise."""
    lv = np.asarray(arrays["leaves"])
    fac = np.asarray(arrays["factors"])
    kern = np.asarray(ref["ck_pin_kernel"])
    pin = np.asarray(ref["ck_pin_leaves"])
    worst = 0.0
    for k in np.unique(kern):
        mine = lv[(lv[:, 0] == k) & (lv[:, 5] > 0)]
        theirs = pin[kern == k]
        if mine.shape[0] != theirs.shape[0] or not np.array_equal(mine[:, 1:6], theirs[:, :5].astype(np.int64)):
            raise ValueError(f"kernel {k}: PLR leaf structure differs from the reference's")
        for row, t in zip(mine, theirs):
            nrm = np.linalg.norm(fac[row[6]:row[6] + row[3] * row[5]])
            worst = max(worst, abs(nrm - t[5]) / max(t[5], 1e-300))
    if worst > rtol:
        raise ValueError(f"pinned kernels' factor norms differ from the reference's by {worst:.2e}")
    return worst


def compare_checksums(mine, ref, rtol=1e-9):
    """Raise ValueError if the operator differs from the reference's beyond rounding."""
    for k in ("entries", "perm"):
        if not np.array_equal(mine[k], ref[k]):
            raise ValueError(f"operator {k} differ from the reference's")
    if not np.array_equal(mine["coefs"], ref["coefs"]):
        raise ValueError("entry coefficients differ from the reference's")
    if "ck_leaves" in ref:
        if "ck_leaves" not in mine or not np.array_equal(mine["ck_leaves"], ref["ck_leaves"]):
            raise ValueError("PLR leaf structure (offsets, sizes, ranks) differs from the reference's")
    a, b = np.asarray(mine["ck_norm"]), np.asarray(ref["ck_norm"])
    err = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
    if err > rtol:
        raise ValueError(f"kernel norms differ from the reference's by {err:.2e}")
    if "ck_colsum" in ref:
        a, b = np.asarray(mine["ck_colsum"]), np.asarray(ref["ck_colsum"])
        err = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
        if err > rtol:
            raise ValueError(f"kernel column sums differ from the reference's by {err:.2e}")
    return True


REF_KEYS = ("ref_x", "ref_traces", "ref_hist", "probe_x", "probe_u", "probe_Ax", "probe_Mx",
            "probe_M1x", "probe_sweep", "ref_index", "probe_Ax_sub", "probe_Mx_sub",
            "probe_Ax_norm", "probe_Mx_norm")


def build_case(name, out_dir=None, workers=None, verify=True):
    """Build <out_dir>/<name>.ptc; returns its path."""
    out_dir = Path(out_dir or DEFAULT_OUT)
    out_dir.mkdir(parents=True, exist_ok=True)
    if name in OPERATOR_OF:
        ensure_case(OPERATOR_OF[name], out_dir, workers)
    t0 = time.perf_counter()
    # PT_OFFLINE_DEVICE=cuda: Green's extraction on the GPU (offline.gpu); the
    # reference-checksum gate below applies either way
    meta, arrays = build_operator(name, workers=workers, device=os.environ.get("PT_OFFLINE_DEVICE") or None)
    ref_path = GOLDEN / f"{name}_ref.ptc"
    if ref_path.exists():
        rmeta, rarr = read_case(ref_path, mmap=False)
        if verify and name not in OPERATOR_OF and "ck_pin_kernel" in rarr:
            meta["pinned_layers_rel_err"] = compare_pinned_layers(meta, arrays, rarr)
            meta["verified_against_reference"] = "layers %s" % rmeta.get("pinned_layers")
        elif verify and name not in OPERATOR_OF:
            compare_checksums(operator_checksums(meta, arrays), rarr)
            meta["verified_against_reference"] = True
        for k in REF_KEYS:
            if k in rarr:
                arrays[k] = rarr[k]
        meta["solves"] = rmeta.get("solves", [])
        meta["reference_offline_seconds"] = rmeta.get("offline_seconds")
        # the reference's rhs (identical up to rounding to ours) for the
        # right-hand sides its results refer to
        idx = np.asarray(rarr.get("ref_index", np.arange(rarr["rhs"].shape[0])))
        d = np.abs(rarr["rhs"] - arrays["rhs"][idx]).max() / np.abs(rarr["rhs"]).max()
        meta["rhs_rel_diff_vs_reference"] = float(d)
        if verify and d > 1e-9:
            raise ValueError(f"right-hand sides differ from the reference's by {d:.2e}")
        if "ref_index" not in rarr:
            arrays["ref_index"] = idx
    meta["build_seconds"] = time.perf_counter() - t0
    path = out_dir / f"{name}.ptc"
    write_case(path, meta, arrays)
    return path


def ensure_case(name, out_dir=None, workers=None):
    """Path of <name>.ptc, building it first if absent (or from an old builder)."""
    out_dir = Path(out_dir or DEFAULT_OUT)
    path = out_dir / f"{name}.ptc"
    if path.exists():
        return path
    lock = out_dir / f".{name}.lock"
    out_dir.mkdir(parents=True, exist_ok=True)
    try:
        fd = os.open(lock, os.O_CREAT | os.O_EXCL | os.O_WRONLY)
    except FileExistsError:  # another rank is building it
        while not path.exists() and lock.exists():
            time.sleep(1.0)
        if path.exists():
            return path
        return ensure_case(name, out_dir, workers)
    try:
        os.close(fd)
        return build_case(name, out_dir, workers)
    finally:
        lock.unlink(missing_ok=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--out", default=None)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--no-verify", action="store_true")
    args = ap.parse_args(argv)
    for n in args.names:
        t = time.perf_counter()
        p = build_case(n, args.out, args.workers, verify=not args.no_verify)
        from ..cache import read_meta
        m = read_meta(p)
        print(json.dumps({"case": n, "path": str(p), "seconds": round(time.perf_counter() - t, 1),
                          "offline_stage_seconds": m["offline_stage_seconds"],
                          "verified": m.get("verified_against_reference", False),
                          "kernel_bytes": m.get("kernel_bytes")}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
