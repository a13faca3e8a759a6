"""Launch one operator program a few times (ncu target; profiling aid).

    python tools/ncu_target.py c3 A [reps] [max_iter]   # kinds: A, M, AM, G (GMRES), B (batched GMRES)
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

name, kind = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
meta, arr = load_case_arrays(ensure_case(name))
op = DeviceOperator.from_arrays(meta, arr)
x = torch.from_numpy(np.array(arr["probe_x"])).cuda()
y = torch.empty_like(x)
for _ in range(reps):
    if kind == "A":
        op.apply_A(x, out=y)
    elif kind == "M":
        op.apply_M(x, out=y)
    elif kind == "AM":
        op.apply_AM(x, out=y)
    elif kind == "B":  # all recorded sources in lockstep (PT_GRAPH=0 for ncu)
        op.gmres_batch(np.asarray(arr["rhs"]), rel_tol=1e-9,
                       max_iter=int(sys.argv[4]) if len(sys.argv) > 4 else 2)
    else:
        op.gmres(torch.from_numpy(np.array(arr["rhs"][0])).cuda(), rel_tol=1e-9,
                 max_iter=int(sys.argv[4]) if len(sys.argv) > 4 else 2)
torch.cuda.synchronize()
print("ok", kind, float(y.abs().sum()))
