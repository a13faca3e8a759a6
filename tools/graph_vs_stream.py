"""Solve time through the graph-resident loop vs the host-driven stream loop (profiling aid).

    python tools/graph_vs_stream.py [case]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
meta, arr = load_case_arrays(ensure_case(name))
op = DeviceOperator.from_arrays(meta, arr)
b = torch.from_numpy(np.array(arr["rhs"][0])).cuda()


def timed(graph, reps=5):
    os.environ["PT_GRAPH"] = "1" if graph else "0"
    for _ in range(2):
        _, rep = op.gmres(b, rel_tol=1e-9, max_iter=100)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        op.gmres(b, rel_tol=1e-9, max_iter=100)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, rep


for g in (True, False, True, False):
    t, rep = timed(g)
    it = rep["iterations"] if isinstance(rep, dict) else rep.iterations
    print(f"{name} graph={g}: {t:.3f} ms per solve, {it} iterations, {t / it * 1e3:.1f} us/iteration")
