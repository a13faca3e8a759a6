"""Critical path of one executor launch (profiling aid, not product code).

    python tools/critical_path.py c3 M [--n 40]

Joins the host plan (pt_plan_tasks: each task's dependency counters) with a
device timeline (pt_trace_program) and walks back from the last task along
the latest-satisfied dependency.  For every task on the path it prints where
the time went: dependency satisfied -> noticed (detect), -> vectors staged,
-> consumers free, -> done.
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
TYPES = {0: "Yd", 1: "Yp", 2: "T"}
TW, TRW = 24, 32  # PT_TASK_WORDS, PT_TRACE_WORDS


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("kind", default="M", nargs="?")
    ap.add_argument("--n", type=int, default=40)
    ap.add_argument("--dump", default=None, help="save the plan and the raw trace (npz)")
    args = ap.parse_args()
    meta, arr = load_case_arrays(ensure_case(args.case))
    op = DeviceOperator.from_arrays(meta, arr)
    k = KIND[args.kind]
    cap = 1 << 20
    plan = np.zeros(cap * TW, dtype=np.int32)
    n = C.c_int64()
    nat.check(nat.lib().pt_plan_tasks(op._h, k, 2, plan.ctypes.data_as(C.POINTER(C.c_int32)), cap,
                                      C.byref(n)))
    plan = plan[: n.value * TW].reshape(n.value, TW)
    x = torch.from_numpy(np.array(arr["probe_x"])).cuda()
    y = torch.empty_like(x)
    rec = np.zeros(cap * TRW, dtype=np.int64)
    for _ in range(2):
        nat.check(nat.lib().pt_trace_program(op._h, k, 2, x.data_ptr(), y.data_ptr(),
                                             rec.ctypes.data_as(C.POINTER(C.c_int64)), cap,
                                             C.byref(n)))
    r = rec[: n.value * TRW].reshape(n.value, TRW)
    if args.dump:
        chain = np.zeros(len(plan), dtype=np.int8)
        np.savez_compressed(args.dump, plan=plan, trace=r)
    t0 = r[:, 6].min()
    us = lambda v: (v - t0) / 1e3  # noqa: E731
    grab, ready, done, cst, staged = us(r[:, 6]), us(r[:, 7]), us(r[:, 8]), us(r[:, 10]), us(r[:, 12])
    # time at which counter c reached value v = v-th done time of its signallers
    by_ctr = {}
    for q in range(len(r)):
        by_ctr.setdefault(int(plan[q, 1]), []).append(done[q])
    for c in by_ctr:
        by_ctr[c].sort()

    def dep_time(q):
        best, arg = 0.0, None
        for i in range(8):
            c, v = int(plan[q, 8 + 2 * i]), int(plan[q, 9 + 2 * i])
            if c < 0 or v <= 0:  # no wait / an empty producer group (dense kernels have no T tasks)
                continue
            if v - 1 >= len(by_ctr.get(c, [])):
                raise SystemExit(f"task {q}: wait ({c}, {v}) but counter has "
                                 f"{len(by_ctr.get(c, []))} signallers; plan rows {len(plan)} "
                                 f"trace rows {len(r)}")
            t = by_ctr[c][v - 1]
            if t > best:
                best, arg = t, c
        return best, arg

    q = int(np.argmax(done))
    path = []
    while q is not None and len(path) < 100000:
        dt, c = dep_time(q)
        path.append((q, dt))
        if c is None:
            break
        # the signaller of counter c that finished last before dt
        cands = [p for p in range(len(r)) if plan[p, 1] == c and abs(done[p] - dt) < 1e-9]
        q = cands[0] if cands else None
    path.reverse()
    print(f"{args.case} {args.kind}: span {done.max():.1f} us, critical path {len(path)} tasks")
    tot = np.zeros(5)
    for q, dt in path:
        seg = np.array([ready[q] - dt, staged[q] - ready[q], cst[q] - staged[q], done[q] - cst[q], 0])
        tot += seg
    print("   sums over the path (us): detect {:.1f} | staging {:.1f} | wait consumers {:.1f} | "
          "compute {:.1f}".format(*tot[:4]))
    print("   q      type pieces  dep_ok  grab-dep  +detect +stage +cons  +busy   done")
    for q, dt in path[: args.n]:
        print(f"   {q:6d} {TYPES.get(int(plan[q, 0]))} {plan[q, 3]:5d} {dt:8.1f} {grab[q] - dt:8.2f} {ready[q] - dt:7.2f} "
              f"{staged[q] - ready[q]:6.2f} {cst[q] - staged[q]:6.2f} {done[q] - cst[q]:6.2f} "
              f"{done[q]:8.1f}")


if __name__ == "__main__":
    main()
