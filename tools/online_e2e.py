"""Whole online stage of solve_helmholtz on the device (profiling aid).

    python tools/online_e2e.py c3 [reps]

restrict + Newton traces + polarized rhs (pt_local_newton), GMRES (pt_gmres),
reconstruction (pt_local_reconstruct); per-stage wall seconds (device
synchronised per stage) next to the reference's own stage seconds recorded
with the case (tests/golden/<case>_ref.ptc, 8-core container).
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200 import solver as S  # noqa: E402
from paper_1410_5910_b200.offline import configs  # noqa: E402
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import load_case_arrays  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
path = ensure_case(name)
meta, arr = load_case_arrays(path)
t0 = time.perf_counter()
state = S.OfflineState.from_case(path, local=True)
setup = time.perf_counter() - t0
f = configs.config(name).sources[0][1]
cfg = S.GmresConfig(rel_tol=meta["gmres_tol"])
rep = S.solve_helmholtz(None, None, None, f, state=state, gmres=cfg)  # warm-up
runs = []
for _ in range(reps):
    rep = S.solve_helmholtz(None, None, None, f, state=state, gmres=cfg)
    runs.append(dict(rep.stage_seconds))
best = {k: min(r[k] for r in runs) for k in runs[0]}
ref = meta["solves"][0].get("stage_seconds", {}) if meta.get("solves") else {}
tr_err = None
if "ref_traces" in arr:
    rt = np.asarray(arr["ref_traces"][0])
    tr_err = float(np.linalg.norm(rep.traces - rt) / np.linalg.norm(rt))
out = {"case": name, "iterations": rep.iterations, "trace_rel_err_vs_reference": tr_err,
       "device_stage_seconds": best, "device_online_seconds": sum(best.values()),
       "reference_stage_seconds": ref,
       "reference_online_seconds": sum(v for k, v in ref.items() if k in
                                       ("restrict", "newton", "rhs", "gmres", "traces", "reconstruct")),
       "local_factor_seconds_host": state.stage_seconds.get("local_factor"),
       "setup_seconds": setup, "local_info": state.local.info}
print(json.dumps(out))
