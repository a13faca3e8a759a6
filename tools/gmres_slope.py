"""Per-iteration cost of the graph-resident GMRES loop (profiling aid).

    python tools/gmres_slope.py c3

Times solves capped at 10 and 30 iterations (CUDA events, warm) and
reports the slope, next to the executor's per-launch time of one fused
A->M iteration program and the Arnoldi kernels from the instrumented path.
"""
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


def timed(k, reps=3):
    op.gmres(b, rel_tol=1e-30, max_iter=k)  # warm / build the graph
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        op.gmres(b, rel_tol=1e-30, max_iter=k)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


t10, t30 = timed(10), timed(30)
print(f"{name}: solve(10 its) {t10:.3f} ms, solve(30 its) {t30:.3f} ms, "
      f"slope {(t30 - t10) / 20 * 1e3:.1f} us/iteration, fixed {t10 - 10 * (t30 - t10) / 20:.3f} ms")
x = torch.from_numpy(np.array(arr["probe_x"])).cuda()
y = torch.empty_like(x)
for _ in range(3):
    op.apply_AM(x, out=y) if hasattr(op, "apply_AM") else None
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    op.apply_AM(x, out=y)
e.record()
torch.cuda.synchronize()
print(f"fused A->M launch (stream, back to back): {s.elapsed_time(e) / 10 * 1e3:.1f} us")
