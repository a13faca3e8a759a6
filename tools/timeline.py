"""Kernel timeline of one graph-resident GMRES solve (profiling aid).

    python tools/timeline.py [case] [out.json]

Runs warm solves, then one solve under torch.profiler (CUPTI kernel
activity, which also records kernels launched from CUDA graph nodes) and
summarises per kernel name: count, mean duration, and the idle gaps between
consecutive device activities (launch boundaries of the per-iteration
graph body: counter memset -> executor -> Arnoldi step).
"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
out = sys.argv[2] if len(sys.argv) > 2 else None
meta, arr = load_case_arrays(ensure_case(name))
op = DeviceOperator.from_arrays(meta, arr)
b = torch.from_numpy(np.array(arr["rhs"][0])).cuda()
for _ in range(3):
    op.gmres(b, rel_tol=1e-9, max_iter=100)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    op.gmres(b, rel_tol=1e-9, max_iter=100)
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    ev.append((e.time_range.start, e.time_range.end, e.name))
ev.sort()
per = defaultdict(list)
gaps = defaultdict(list)
for i, (s, t, n) in enumerate(ev):
    short = n.replace("(anonymous namespace)::", "").split("(")[0].replace("pt::", "")[:60]
    per[short].append(t - s)
    if i:
        prev = ev[i - 1][2].replace("(anonymous namespace)::", "").split("(")[0].replace("pt::", "")[:40]
        gaps[f"{prev} -> {short[:40]}"].append(s - ev[i - 1][1])
summary = {
    "case": name,
    "span_us": ev[-1][1] - ev[0][0] if ev else 0,
    "kernels": {k: {"n": len(v), "mean_us": float(np.mean(v)), "total_us": float(np.sum(v))}
                for k, v in per.items()},
    "gaps": {k: {"n": len(v), "mean_us": float(np.mean(v)), "total_us": float(np.sum(v))}
             for k, v in gaps.items()},
}
print(json.dumps(summary, indent=1))
if out:
    Path(out).write_text(json.dumps(summary, indent=1))
