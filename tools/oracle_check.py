"""Parity of the device GMRES against the oracle port on one case (test aid).

    python tools/oracle_check.py c4 [--out gpurun_out/c4_parity.json]

For cases with no reference solve recorded (c4: the reference's own offline
stage takes hours here), the oracle (oracle/ref_port.py, pinned to the
reference on c1-c3/c5) is the checker: same operator, same right-hand side,
MGS + lstsq GMRES on the host.  Reports iterations and the relative L2
difference of the traces u = x_down + x_up.
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import ref_port as O  # noqa: E402
from paper_1410_5910_b200.offline.build import ensure_case  # noqa: E402
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    meta, arr = load_case_arrays(ensure_case(args.case))
    tol, mx, n_it = meta["gmres_tol"], meta["gmres_max_iter"], meta["n_it"]
    b = np.array(arr["rhs"][0])
    op = DeviceOperator.from_arrays(meta, arr)
    xg, rg = op.gmres(torch.from_numpy(b).cuda(), rel_tol=tol, max_iter=mx, n_it=n_it)
    xg = xg.cpu().numpy()
    t0 = time.perf_counter()
    pol, perm = O.operator_from_case(meta, arr)
    d, r = O.split_dr(pol, perm)
    t1 = time.perf_counter()
    xo, ro = O.gmres_solve(pol.matvec, lambda v: O.preconditioner_apply(n_it, d, r, perm, v), b,
                           rel_tol=tol, max_iter=mx)
    t2 = time.perf_counter()
    nt, m = meta["nt"], meta["m"]
    tg, to = xg[: nt * m] + xg[nt * m:], xo[: nt * m] + xo[nt * m:]
    res = {
        "case": args.case, "N": int(b.size), "gpu_iterations": int(rg["iterations"]),
        "oracle_iterations": int(ro.iterations), "gpu_flag": rg["flag"],
        "trace_rel_l2_vs_oracle": float(np.linalg.norm(tg - to) / np.linalg.norm(to)),
        "x_rel_l2_vs_oracle": float(np.linalg.norm(xg - xo) / np.linalg.norm(xo)),
        "oracle_setup_s": t1 - t0, "oracle_gmres_s": t2 - t1,
    }
    print(json.dumps(res))
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
