"""One warm device GMRES solve on a case (driver for ncu captures; PT_GRAPH=0 for per-kernel launches)."""
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
for _ in range(2):
    _, rep = op.gmres(b, rel_tol=1e-9, max_iter=100)
torch.cuda.synchronize()
print(name, rep["iterations"])
