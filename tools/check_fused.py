"""Debug aid: fused A->M program vs separate A then M applies, repeatability."""
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

for name in sys.argv[1:]:
    path = ROOT / "tests" / "golden" / f"{name}.ptc" if name.startswith("fx") else ensure_case(name)
    meta, arr = load_case_arrays(path)
    op = DeviceOperator.from_arrays(meta, arr)
    x = torch.from_numpy(np.array(arr["probe_x"])).cuda()
    ref = op.apply_M(op.apply_A(x))
    cap = 1 << 20
    rec = np.zeros(cap * 32, dtype=np.int64)
    n = C.c_int64()
    errs = []
    for rep in range(6):
        y = torch.empty_like(x)
        rc = nat.lib().pt_trace_program(op.handle, 2, 2, x.data_ptr(), y.data_ptr(),
                                        rec.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(n))
        nat.check(rc)
        errs.append(float((y - ref).abs().max() / ref.abs().max()))
    a1 = op.apply_A(x)
    a_err = [float((op.apply_A(x) - a1).abs().max()) for _ in range(5)]
    m1 = op.apply_M(x)
    m_err = [float((op.apply_M(x) - m1).abs().max()) for _ in range(5)]
    print(name, "fused AM vs A;M:", ["%.1e" % e for e in errs], "A repeat:", max(a_err),
          "M repeat:", max(m_err), op.exec_info(), flush=True)
