"""Quick device timing of applies and a GMRES solve on available cases (dev aid)."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402

PEAK = 6540.2


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for name in sys.argv[1:]:
    if name.startswith("fx_"):
        path = ROOT / "tests" / "golden" / f"{name}.ptc"
    else:
        from paper_1410_5910_b200.offline.build import ensure_case
        path = ensure_case(name)
    if not path.exists():
        print(name, "missing")
        continue
    t0 = time.perf_counter()
    meta, arr = load_case_arrays(path)
    op = DeviceOperator.from_arrays(meta, arr)
    t_up = time.perf_counter() - t0
    x = torch.from_numpy(np.asarray(arr["probe_x"])).cuda()
    y = torch.empty_like(x)
    bA, bM = op.bytes_apply_A(), op.bytes_apply_M(2)
    tA = timed(lambda: op.apply_A(x, out=y))
    tM = timed(lambda: op.apply_M(x, n_it=2, out=y))
    b = torch.from_numpy(np.asarray(arr["rhs"][0])).cuda()
    xo = torch.empty_like(b)
    op.gmres(b, rel_tol=meta["gmres_tol"], out=xo)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, rep = op.gmres(b, rel_tol=meta["gmres_tol"], out=xo)
    torch.cuda.synchronize()
    tg = (time.perf_counter() - t1) * 1e3
    k = rep["iterations"]
    print(f"{name}: m={meta['m']} L={meta['L']} fmt={op.kernel_format} upload {t_up:.1f}s | "
          f"A {tA*1e3:.1f} us {bA/tA/1e6:.0f} GB/s ({bA/tA/1e6/PEAK:.2f}) | "
          f"M {tM*1e3:.1f} us {bM/tM/1e6:.0f} GB/s ({bM/tM/1e6/PEAK:.2f}) | "
          f"gmres {tg:.2f} ms it={k} ref_it={meta['solves'][0]['iterations']} "
          f"per-it {tg/max(k,1):.3f} ms {op.exec_info()}",
          flush=True)
    op.close()
