#!/usr/bin/env python
"""Benchmark: online polarized-traces GMRES solve on B200 (one JSON line).

A "step" is one full online GMRES solve (the "gmres" stage of the
reference's solve_helmholtz, solver.py:376-397) of one right-hand side on the
BASELINE configuration c3 (n=800^2 + 40 PML, L=16, layered medium, PLR
operators) -- the configuration BASELINE.json's metric is quoted on.  The
operator comes from the PTC1 cache built by the reference's own offline
stage (tools/make_cases.py); it is uploaded to HBM before timing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
  python bench.py --impl reference ...      # CPU reference arm (oracle port)

N > 1 runs under torchrun as independent replicas (the path
does not shard; no collective on the data path), timed as the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "online solve ms & trace-apply HBM GB/s (fraction of peak), n=800², L=16"
DATA = ("synthetic (seeded media per SURVEY.md §8(d)); operator built on this host by the restated "
        "reference offline stage and verified against the reference's own checksums")
# FP64 tensor-core peak of one B200 measured with tools/dmma_bench.cu
# (profiles/r01_fp64_dmma_vs_dfma.txt; mma.sync m8n8k4/m16n8k16 .f64)
FP64_TENSOR_TFLOPS = 36.9
FP64_PEAK_SRC = "measured (tools/dmma_bench.cu, profiles/r01_fp64_dmma_vs_dfma.txt)"
FALLBACK_HBM = 6650.0
L2_BYTES = 126 * 2**20
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="case name (default: c3, else c2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-online", action="store_true",
                    help="skip the whole-online-stage line (Newton + GMRES + reconstruction)")
    return ap.parse_args()


def pick_case(name):
    """The workload's PTC1 operator cache, built by the host offline stage if absent.

    The c3 operator (626 MB) exceeds what ships to the GPU box; it is rebuilt
    there by the restated reference offline stage (layer-parallel, ~2-3 min on
    16 cores) and verified against the reference's checksums
    (tests/golden/c3_ref.ptc), then reused from $PT_CASES (default cases/).
    """
    from paper_1410_5910_b200.offline.build import ensure_case
    name = name or "c3"
    t0 = time.perf_counter()
    path = ensure_case(name)
    dt = time.perf_counter() - t0
    if dt > 1.0:
        print(f"[bench] built {path} in {dt:.0f} s (host offline stage, not timed)",
              file=sys.stderr, flush=True)
    return name, path


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def workload_config(name, meta, extra=None):
    cfg = {
        "workload": f"{name}: {meta['note']}",
        "case": name,
        "nx": meta["nx"], "nz": meta["nz"], "n_pml": meta["n_pml"], "L": meta["L"],
        "m": meta["m"], "unknowns": 2 * meta["nt"] * meta["m"],
        "omega": round(meta["omega"], 4),
        "kernel_format": meta.get("kernel_format"),
        "kernel_bytes": meta.get("kernel_bytes"),
        "gmres_tol": meta["gmres_tol"], "max_iter": meta["gmres_max_iter"], "n_it": meta["n_it"],
        "rhs": meta["solves"][0]["label"] if meta.get("solves") else "rhs[0] (point source)",
        "l2": "flushed between steps (256 MiB write); operator %.0f MB vs 126 MB L2"
              % (meta.get("kernel_bytes", 0) / 1e6),
        "parallelism": "replicas",
    }
    if extra:
        cfg.update(extra)
    return cfg


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the timed region runs."""

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_id),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m_ = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            sm.append(s)
            mx.append(m_)
            for bit, name in REASONS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(backend):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and backend:
        import torch.distributed as dist
        dist.init_process_group(backend)
    return world, rank, local


# ----------------------------------------------------------------------------
# CPU side: the oracle port (test/baseline infrastructure; never the product)


_ORACLE = {}


def cpu_sample(meta, arr):
    """Time one full oracle GMRES solve of rhs[0] (M-apply of b, every
    iteration to convergence, the true-residual A-apply), in ms."""
    from oracle import ref_port as O
    key = meta["name"]
    if key not in _ORACLE:  # built once, outside the timed sample
        pol, perm = O.operator_from_case(meta, arr)
        _ORACLE[key] = (pol, perm, O.split_dr(pol, perm))
    pol, perm, (d, r) = _ORACLE[key]
    b = np.asarray(arr["rhs"][0])
    M = lambda v: O.preconditioner_apply(meta["n_it"], d, r, perm, v)  # noqa: E731
    t0 = time.perf_counter()
    _, rep = O.gmres_solve(pol.matvec, M, b, rel_tol=meta["gmres_tol"], max_iter=meta["gmres_max_iter"])
    return (time.perf_counter() - t0) * 1e3, rep


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count()


def run_reference(args):
    world, rank, local = dist_setup(None)
    if rank != 0:
        return
    name, path = pick_case(args.config)
    from paper_1410_5910_b200.operator import load_case_arrays
    meta, arr = load_case_arrays(path)
    # every step is one full solve (no extrapolation): ~13 s at c3 on 16 cores
    for _ in range(args.warmup):
        cpu_sample(meta, arr)
    vals, its = [], []
    for _ in range(args.steps):
        v, rep = cpu_sample(meta, arr)
        vals.append(v)
        its.append(rep.iterations)
    value = float(np.mean(vals))
    cores = cpu_threads()
    sample = (f"oracle port of gmres_solve (MGS + lstsq, numpy/OpenBLAS + scipy CSR) on {name}: "
              f"one full solve of rhs[0] per step ({its[0]} iterations, to convergence), "
              f"mean of {args.steps} after {args.warmup} warm-up solves")
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128", "data": DATA,
        "config": workload_config(name, meta), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "ms", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------


def online_pipeline(name, meta, op, device, tol):
    """The whole online stage of solve_helmholtz on the device (restrict,
    Newton traces + polarized rhs, GMRES, reconstruction),
    best of 3 after a warm-up, next to the reference's own host stage seconds
    recorded with the case.  Reported beside the metric, not part of it."""
    import torch
    from paper_1410_5910_b200 import solver as S
    from paper_1410_5910_b200.local import DeviceLocalSolver
    from paper_1410_5910_b200.offline.configs import config as case_config
    t0 = time.perf_counter()
    loc = DeviceLocalSolver.from_config(name, device=device)
    factor_s = time.perf_counter() - t0
    state = S.OfflineState(op=op, variant=meta.get("variant", "jump"), meta=meta, local=loc)
    f = case_config(name).sources[0][1]
    cfg = S.GmresConfig(rel_tol=tol)
    runs = []
    for _ in range(4):
        rep = S.solve_helmholtz(None, None, None, f, state=state, gmres=cfg)
        runs.append(rep.stage_seconds)
    best = {k: min(r[k] for r in runs[1:]) * 1e3 for k in runs[0]}
    ref = (meta.get("solves") or [{}])[0].get("stage_seconds", {})
    ref_ms = {k: v * 1e3 for k, v in ref.items()
              if k in ("restrict", "newton", "rhs", "gmres", "reconstruct")}
    out = {"device_stage_ms": best, "device_total_ms": sum(best.values()),
           "iterations": rep.iterations, "local_factor_host_s": factor_s,
           "local_levels": loc.info["l_levels"],
           "reference_host_stage_ms": ref_ms or None,
           "reference_host_total_ms": sum(ref_ms.values()) if ref_ms else None,
           "note": "per-stage wall time, device synchronised per stage; reference stage "
                   "seconds recorded with the case (8-core container)"}
    loc.close()
    torch.cuda.synchronize(device)
    return out


def run_ours(args):
    import torch
    world, rank, local = dist_setup("nccl" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else None)
    torch.cuda.set_device(local)
    from paper_1410_5910_b200 import _native
    from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays

    name, path = pick_case(args.config)
    meta, arr = load_case_arrays(path)
    t0 = time.perf_counter()
    op = DeviceOperator.from_arrays(meta, arr, device=local)
    upload_s = time.perf_counter() - t0
    N = op.N
    tol, max_iter, n_it = meta["gmres_tol"], meta["gmres_max_iter"], meta["n_it"]
    from paper_1410_5910_b200.replicas import gather_counts, max_over_ranks, shard
    nrhs = int(np.asarray(arr["rhs"]).shape[0])
    # multi-RHS workloads shard their sources across ranks; single-RHS ones
    # run one replica per rank (no collective on the data path)
    mine = list(shard(nrhs, world, rank)) if nrhs > 1 else [0]
    rhs_dev = [torch.from_numpy(np.array(arr["rhs"][s])).to(f"cuda:{local}") for s in mine]
    b = rhs_dev[0]
    x = torch.empty_like(b)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    # multi-source dense workloads (c5) run the sources in lockstep batches on
    # the batched executor (pt_gmres_batch); single sources the fused path
    batched = (len(mine) > 1 and meta.get("kernel_format") == "dense"
               and not os.environ.get("PT_BATCH_SEQ"))
    B_dev = torch.stack(rhs_dev) if batched else None

    def step():
        """One step; returns the report of every solve in it."""
        if batched:
            _, reps = op.gmres_batch(B_dev, rel_tol=tol, max_iter=max_iter, n_it=n_it)
            return list(reps)
        out = []
        for bs in rhs_dev:
            _, rep = op.gmres(bs, rel_tol=tol, max_iter=max_iter, n_it=n_it, out=x)
            out.append(rep)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    gpu_uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    barrier()
    lib = _native.lib()
    launches0 = lib.pt_launch_count()
    step_ms, reps = [], []
    with ClockSampler(gpu_uuid) as clk:
        for _ in range(args.steps):
            flush.zero_()  # evict L2 (outside the timed interval)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            reps.extend(rep)
    launches = lib.pt_launch_count() - launches0
    barrier()
    total_ms = float(sum(step_ms))

    # roofline of the dominant kernel: the same K solves again with every
    # executor launch bracketed by CUDA events on its stream (host-driven
    # launch path; the kernel is the same one the graph replays)
    op.exec_timing(True)
    instr_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        instr_ms.append(e0.elapsed_time(e1))
    exec_ms, exec_n, exec_bytes = op.exec_stats()
    op.exec_timing(False)
    instr_total = float(sum(instr_ms))

    # end to end through the host-buffer C-ABI call (pt_gmres_host): H2D of b
    # from pinned memory, the solve, D2H of x, all inside the timed interval
    b_host = [torch.from_numpy(np.array(arr["rhs"][s])).pin_memory() for s in mine]
    x_host = torch.empty_like(b_host[0]).pin_memory()
    e2e_ms = []

    B_host = torch.stack(b_host).pin_memory() if batched else None
    X_host = torch.empty_like(B_host).pin_memory() if batched else None

    def step_host():
        if batched:
            op.gmres_batch_host(B_host, X_host, rel_tol=tol, max_iter=max_iter, n_it=n_it)
            return
        for bh in b_host:
            op.gmres_host(bh, x_host, rel_tol=tol, max_iter=max_iter, n_it=n_it)

    step_host()
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step_host()
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_total = float(sum(e2e_ms))
    dev = f"cuda:{local}"
    total_ms = max_over_ranks(total_ms, dev)
    e2e_total = max_over_ranks(e2e_total, dev)
    solves_per_step = gather_counts(len(mine), dev)

    # parity vs the reference's own solution of its first recorded right-hand
    # side (c5 records a subset, ref_index), solved again after the timing
    nt, m = meta["nt"], meta["m"]
    ri = int(np.asarray(arr["ref_index"])[0]) if "ref_index" in arr else 0
    b_chk = torch.from_numpy(np.array(arr["rhs"][ri])).to(f"cuda:{local}")
    x_chk, rep_chk = op.gmres(b_chk, rel_tol=tol, max_iter=max_iter, n_it=n_it)
    xs = x_chk.cpu().numpy() if hasattr(x_chk, "cpu") else np.asarray(x_chk)
    if "ref_traces" in arr:
        ref_tr = np.asarray(arr["ref_traces"][0])
        trace_err = float(np.linalg.norm(xs[:nt * m] + xs[nt * m:] - ref_tr) / np.linalg.norm(ref_tr))
    else:  # no reference solve for this case (c4: see DESIGN.md, parity vs the oracle)
        trace_err = None
    k = rep_chk["iterations"]

    online = None
    if world == 1 and not batched and not args.no_online:
        online = online_pipeline(name, meta, op, local, tol)

    ref_k = meta["solves"][0]["iterations"] if meta.get("solves") else None
    all_conv = all(bool(r.get("converged")) for r in reps) and bool(rep_chk.get("converged"))
    invalid = []  # the gates smoke() and the tests use
    if not all_conv:
        invalid.append("a timed solve did not converge")
    if ref_k is not None and abs(k - ref_k) > 1:
        invalid.append(f"iterations {k} vs reference {ref_k}")
    if trace_err is not None and not trace_err <= 1e-8:
        invalid.append(f"trace error {trace_err:.3e} > 1e-8")

    if rank != 0:
        return
    peak, peak_src = peaks()
    achieved = exec_bytes / (exec_ms * 1e-3) / 1e9 if exec_ms > 0 else None
    roof_unit, bound = "GB/s", "hbm"
    if batched:
        # FP64-tensor-bound: 8 flop per kernel element per source;
        # peak = the mma.sync .f64 rate measured on this GPU (no FP64 entry in
        # MEASURED_PEAKS.json)
        per_batch = min(len(mine), 64)
        flops = exec_bytes / 16 * 8 * per_batch
        achieved = flops / (exec_ms * 1e-3) / 1e12 if exec_ms > 0 else None
        peak, peak_src = FP64_TENSOR_TFLOPS, FP64_PEAK_SRC
        roof_unit, bound = "TFLOP/s", "tensor"
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(name)
    per_step_bytes = exec_bytes / max(args.steps * len(mine), 1)  # algorithmic bytes per solve
    value = total_ms / (args.steps * solves_per_step)
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128",
        "data": DATA,
        "config": workload_config(name, meta),
        "parity": {"iterations": k,
                   "reference_iterations": ref_k,
                   "trace_rel_err_vs_reference": trace_err,
                   "timed_solves_converged": all_conv,
                   "sources": len(mine),
                   "batched": ("lockstep batches of 64 (pt_gmres_batch)" if batched else None)},
        "impl": "ours",
        "roofline": {
            "bound": bound, "achieved": achieved, "peak": peak, "unit": roof_unit,
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "kernel": ("pt_bexec_kernel (batched A->M iteration program, DMMA)" if batched else
                       "pt_exec_kernel (operator applies: fused A->M iteration program)"),
            "algorithmic_bytes_per_launch": exec_bytes / max(exec_n, 1),
            "launch_ms_avg": exec_ms / max(exec_n, 1), "launches": exec_n,
            "peak_source": peak_src,
            "kernel_share_of_step": exec_ms / instr_total if instr_total > 0 else None,
            "measured": "per-launch CUDA events in an instrumented pass of the same K solves",
        },
        "solve": {"per_iteration_ms": (total_ms / args.steps / len(mine)) / max(k, 1),
                  "solves_per_step": solves_per_step,
                  "solve_gbs": per_step_bytes / (total_ms / args.steps / len(mine) * 1e-3) / 1e9,
                  # solve-level fraction in the roofline's own unit: HBM bytes per
                  # solve time, or (batched) the lockstep batch's flops per step time
                  "solve_frac": ((exec_bytes / 16 * 8 * min(len(mine), 64)) / (total_ms * 1e-3) / 1e12
                                 / peak if batched else
                                 per_step_bytes / (total_ms / args.steps / len(mine) * 1e-3) / 1e9
                                 / peak),
                  "algorithmic_bytes_per_solve": per_step_bytes,
                  "upload_s": upload_s, "offline_host_s": meta.get("offline_seconds")},
        "e2e": {"value": e2e_total / (args.steps * solves_per_step), "unit": "ms",
                "h2d_bytes_per_step": N * 16 * len(mine), "d2h_bytes_per_step": N * 16 * len(mine),
                "api": ("pt_gmres_batch_host" if batched else "pt_gmres_host")
                       + " (C ABI, pinned host b/x)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if online is not None:
        line["online_pipeline"] = online
    if world == 1 and not args.no_cpu_baseline:
        cpu_ms, cpu_rep = cpu_sample(meta, arr)
        line["cpu_baseline"] = {
            "value": cpu_ms, "unit": "ms", "cores": cpu_threads(), "kind": "port",
            "sample": f"one full oracle gmres_solve of rhs[0] on {name} ({cpu_rep.iterations} "
                      f"iterations, to convergence); numpy/OpenBLAS threads = cores, scipy CSR "
                      f"single-threaded",
        }
    if invalid:
        line["invalid"] = "; ".join(invalid)
        print(json.dumps(line), flush=True)
        sys.exit(3)
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
