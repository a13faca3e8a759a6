"""Build (if needed) and time one case on the device (dev aid; no reference needed).

    python tools/case_probe.py c4
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

name = sys.argv[1]
t0 = time.perf_counter()
path = ensure_case(name)
print(f"{name}: case ready in {time.perf_counter() - t0:.0f} s ({path.stat().st_size / 1e9:.2f} GB)",
      flush=True)
meta, arr = load_case_arrays(path)
op = DeviceOperator.from_arrays(meta, arr)
print(f"  m={meta['m']} nt={meta['nt']} N={op.N} format={op.kernel_format} info={op.exec_info()} "
      f"A bytes={op.bytes_apply_A() / 1e6:.1f} MB M2 bytes={op.bytes_apply_M(2) / 1e6:.1f} MB", flush=True)
b = torch.from_numpy(np.array(arr["rhs"][0])).cuda()
x, rep = op.gmres(b, rel_tol=meta["gmres_tol"], max_iter=meta["gmres_max_iter"])
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    x, rep = op.gmres(b, rel_tol=meta["gmres_tol"], max_iter=meta["gmres_max_iter"])
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
print(f"  gmres {ms:.2f} ms, {rep['iterations']} iterations, flag {rep['flag']}, "
      f"true residual {rep['true_residual']:.2e}", flush=True)
