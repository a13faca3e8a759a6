"""Per-task timeline of one executor launch (profiling aid, not product code).

    python tools/trace_exec.py c3 [AM|A|M] [--out gpurun_out/trace_c3.npz]

Uses pt_trace_program: every task records the globaltimer when its CTA
grabbed it, when its dependencies were satisfied and when it finished.
Prints where the launch spends its time: per task type busy time, waits,
and an occupancy profile over the launch.
"""

import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200 import _native as nat  # noqa: E402
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

KIND = {"A": 0, "M": 1, "AM": 2, "S": 3}
TYPES = {0: "Ydense", 1: "Yplr", 2: "Tplr"}
W = 32  # PT_TRACE_WORDS


def trace(op, kind, x, n_it=2):
    y = torch.empty_like(x)
    cap = 1 << 20
    rec = np.zeros(cap * W, dtype=np.int64)
    n = C.c_int64()
    rc = nat.lib().pt_trace_program(op.handle, KIND[kind], n_it, x.data_ptr(), y.data_ptr(),
                                    rec.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(n))
    nat.check(rc, "trace")
    return rec[: n.value * W].reshape(n.value, W)


def summarize(r, label):
    t0 = r[:, 6].min()
    grab, ready, done = (r[:, 6] - t0) / 1e3, (r[:, 7] - t0) / 1e3, (r[:, 8] - t0) / 1e3
    span = done.max()
    print(f"== {label}: {len(r)} tasks, launch span {span:.1f} us")
    p0 = np.where(r[:, 10] > 0, (r[:, 10] - t0) / 1e3, np.nan)
    for ty in sorted(set(r[:, 0])):
        sel = r[:, 0] == ty
        busy = (done - ready)[sel]
        wait = (ready - grab)[sel]
        # time after the dependency wait until the first operator piece was in smem
        pw = np.nanmean(np.maximum(p0[sel] - ready[sel], 0)) if np.isfinite(p0[sel]).any() else 0
        # piece-0 latency from issue (grab) to arrival
        pl = np.nanmean(p0[sel] - grab[sel]) if np.isfinite(p0[sel]).any() else 0
        print(f"  {TYPES.get(int(ty), ty):7s} n={sel.sum():5d} busy mean {busy.mean():6.2f} us "
              f"max {busy.max():6.2f}  sum {busy.sum():9.1f} | wait mean {wait.mean():6.2f} "
              f"max {wait.max():6.2f} | piece0 arrives {pl:5.2f} after grab, "
              f"{pw:5.2f} after ready")
    nbins = 40
    edges = np.linspace(0, span, nbins + 1)
    act = []
    for a, b in zip(edges[:-1], edges[1:]):
        act.append(int(((ready < b) & (done > a)).sum()))
    print("  computing tasks over time (40 bins):", act)
    # groups = output blocks (signal counters): their completion times
    grp = {}
    for q in range(len(r)):
        g = int(r[q, 11])
        grp.setdefault(g, []).append(q)
    ends = sorted((done[qs].max(), g, len(qs), TYPES.get(int(r[qs[0], 0]))) for g, qs in grp.items())
    print(f"  {len(grp)} producer groups; completion times of the last 12:")
    for e, g, n, ty in ends[-12:]:
        print(f"    group {g:4d} {ty:6s} tasks {n:3d} done at {e:8.1f} us")
    return span


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("kinds", nargs="*", default=["A", "M", "AM"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    meta, arr = load_case_arrays(ensure_case(args.case) if not args.case.startswith("fx_")
                                 else ROOT / "tests" / "golden" / f"{args.case}.ptc")
    op = DeviceOperator.from_arrays(meta, arr)
    x = torch.from_numpy(np.array(arr["probe_x"])).cuda()
    res = {}
    for k in args.kinds:
        trace(op, k, x)  # warm
        r = trace(op, k, x)
        summarize(r, f"{args.case} {k}")
        phases(r, f"{args.case} {k}")
        res[k] = r
    if args.out:
        np.savez(args.out, **res)




def phases(r, label):
    """Mean in-task phase durations (us) per task type from the marks."""
    print(f"-- {label} in-task phases (mean us)")
    us = lambda a, b: np.where((a > 0) & (b > 0), (a - b) / 1e3, np.nan)  # noqa: E731
    for ty in sorted(set(r[:, 0])):
        rr = r[r[:, 0] == ty]
        ready, staged, cstart, done = rr[:, 7], rr[:, 12], rr[:, 10], rr[:, 8]
        issue, landed = rr[:, 14:22], rr[:, 22:30]
        lat = np.nanmean(us(landed, issue))
        gaps = np.nanmean(us(landed[:, 1:], landed[:, :-1]))
        pre = np.nanmean(np.where(issue[:, 0] > 0, (issue[:, 0] < ready), np.nan))
        print(f"   {TYPES.get(int(ty), ty):7s} pieces {rr[:, 13].mean():5.1f} | ready->staged "
              f"{np.nanmean(us(staged, ready)):5.2f} | staged->consumers "
              f"{np.nanmean(us(cstart, staged)):5.2f} | consumers busy {np.nanmean(us(done, cstart)):5.2f} "
              f"| piece issue->seen {lat:5.2f} | gap between pieces seen {gaps:5.2f} | "
              f"piece0 issued before ready {pre:4.2f} | consumer cycles: wait pieces "
              f"{rr[:, 30].mean():7.0f} barrier {rr[:, 31].mean():7.0f} "
              f"(of {np.nanmean(us(done, cstart)) * 1.9e3:7.0f})")


if __name__ == "__main__":
    main()
