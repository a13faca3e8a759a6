"""Per-CTA view of a trace_exec.py capture (profiling aid).

    python tools/trace_cta.py gpurun_out/trace_c3.npz [A M AM]

For every CTA, walks its tasks in queue order and splits the launch into
consumer busy time, consumer idle time and, for the idle part, what the
producer warp was doing (metadata, dependency wait, staging).
"""
import sys

import numpy as np


def analyse(r, label):
    r = r.astype(np.int64)
    t0 = r[:, 6].min()
    cta = r[:, 9] >> 16
    grab, ready, done, cst, staged = [(r[:, i] - t0) / 1e3 for i in (6, 7, 8, 10, 12)]
    span = done.max()
    ncta = len(np.unique(cta))
    idle, busy, dep, meta, stg = [], [], [], [], []
    for c in np.unique(cta):
        qs = np.where(cta == c)[0]
        prev_done = 0.0
        for q in qs:
            idle.append(max(cst[q] - prev_done, 0))
            busy.append(done[q] - cst[q])
            stg.append(staged[q] - ready[q])
            prev_done = done[q]
    idle, busy, stg = map(np.array, (idle, busy, stg))
    print(f"== {label}: span {span:.1f} us, {ncta} CTAs, {len(r) / ncta:.1f} tasks/CTA")
    print(f"   consumer busy {busy.sum() / ncta:6.1f} us/CTA ({busy.sum() / ncta / span:4.0%}), "
          f"idle {idle.sum() / ncta:6.1f} us/CTA")
    types = {0: "Ydense", 1: "Yplr", 2: "Tplr"}
    for ty in sorted(set(r[:, 0])):
        sel = r[:, 0] == ty
        print(f"   {types.get(int(ty), ty):7s} n={sel.sum():6d} busy {busy[sel].mean():5.2f} us "
              f"(sum/CTA {busy[sel].sum() / ncta:6.1f}) | grab->ready {(ready - grab)[sel].mean():5.2f} "
              f"| staging {stg[sel].mean():5.2f} | bytes/piece-seq gap n/a")
    # time profile of how many consumers are busy
    edges = np.linspace(0, span, 21)
    prof = [int(((cst < b) & (done > a)).sum()) for a, b in zip(edges[:-1], edges[1:])]
    print("   busy CTAs over time:", prof)


if __name__ == "__main__":
    d = np.load(sys.argv[1])
    for k in (sys.argv[2:] or d.files):
        analyse(d[k], k)
