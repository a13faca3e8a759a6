"""Small workload for compute-sanitizer (profiling aid): every executor
program, the Arnoldi step and the batched executor on tiny fixtures.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py fx_plr
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

for name in sys.argv[1:]:
    meta, arr = load_case_arrays(ROOT / "tests" / "golden" / f"{name}.ptc")
    op = DeviceOperator.from_arrays(meta, arr)
    x = torch.from_numpy(np.array(arr["probe_x"])).cuda()
    u = torch.from_numpy(np.array(arr["probe_u"])).cuda()
    ya, zm, zam = op.apply_A(x), op.apply_M(x, n_it=2), op.apply_AM(x, n_it=2)
    zs = op.gs_sweep(x, u)
    b = torch.from_numpy(np.array(arr["rhs"][0])).cuda()
    xs, rep = op.gmres(b, rel_tol=meta["gmres_tol"], max_iter=8)
    msg = f"{name}: A {float(ya.abs().sum()):.6e} M {float(zm.abs().sum()):.6e} " \
          f"AM {float(zam.abs().sum()):.6e} S {float(zs.abs().sum()):.6e} gmres it {rep['iterations']}"
    if op.kernel_format == "dense":  # the batched executor (c5's path)
        B = torch.stack([b, x, u, b + x]).contiguous()
        Xb, reps = op.gmres_batch(B, rel_tol=meta["gmres_tol"], max_iter=6)
        msg += f" batch its {[r['iterations'] for r in reps]}"
    torch.cuda.synchronize()
    print(msg, flush=True)
    op.close()
