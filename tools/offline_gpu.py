"""Offline stage on the GPU vs on the host workers (profiling aid).

    python tools/offline_gpu.py c3 [--workers 16] [--layers 4]

Builds the operator of a case with the Green's extraction and the PLR
compression on the GPU (offline.gpu) and prints the stage times next to the
host build's; --layers N times only the first N layers of each.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1410_5910_b200.offline import build as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--host", action="store_true", help="also time the host build")
    ap.add_argument("--compress-on", default="host", choices=["host", "cuda"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    torch.cuda.init()
    res = {"case": args.case, "compress_on": args.compress_on}
    t0 = time.perf_counter()
    m_g, a_g = B.build_operator(args.case, workers=args.workers, sources=True, device="cuda",
                                compress_on=args.compress_on)
    res["gpu"] = {"wall_s": time.perf_counter() - t0, "stage_s": m_g["offline_stage_seconds"],
                  "workers": m_g["offline_workers"]}
    print("gpu ", json.dumps(res["gpu"]))
    if args.host:
        t0 = time.perf_counter()
        m_h, a_h = B.build_operator(args.case, workers=args.workers, sources=True)
        res["host"] = {"wall_s": time.perf_counter() - t0, "stage_s": m_h["offline_stage_seconds"],
                       "workers": m_h["offline_workers"]}
        print("host", json.dumps(res["host"]))
        if "leaves" in a_h:
            same = a_h["leaves"].shape == a_g["leaves"].shape and np.array_equal(a_h["leaves"], a_g["leaves"])
            res["leaf_tables_equal"] = bool(same)
            res["leaves"] = [int(a_h["leaves"].shape[0]), int(a_g["leaves"].shape[0])]
        else:
            res["dense_rel_diff"] = float(np.linalg.norm(a_h["dense"] - a_g["dense"]) / np.linalg.norm(a_h["dense"]))
        res["rhs_rel_diff"] = float(np.linalg.norm(a_h["rhs"] - a_g["rhs"]) / np.linalg.norm(a_h["rhs"]))
        print({k: res[k] for k in res if k not in ("gpu", "host")})
    # the reference's own checksums of this operator (tests/golden/<case>_ref.ptc)
    ref_path = B.GOLDEN / f"{args.case}_ref.ptc"
    if ref_path.exists():
        rmeta, rarr = B.read_case(ref_path, mmap=False)
        try:
            if "ck_pin_kernel" in rarr:
                res["gpu_vs_reference"] = B.compare_pinned_layers(m_g, a_g, rarr)
            else:
                B.compare_checksums(B.operator_checksums(m_g, a_g), rarr)
                res["gpu_vs_reference"] = "checksums equal (leaf structure identical, norms within 1e-9)"
        except Exception as exc:  # noqa: BLE001
            res["gpu_vs_reference"] = f"MISMATCH: {exc}"
        print("gpu build vs the reference's checksums:", res["gpu_vs_reference"])
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
