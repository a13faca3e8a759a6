import sys, numpy as np
sys.path.insert(0, ".")
from paper_1410_5910_b200.offline.build import ensure_case
from paper_1410_5910_b200.operator import DeviceOperator, load_case_arrays
meta, arr = load_case_arrays(ensure_case("c4"))
op = DeviceOperator.from_arrays(meta, arr)
rel = lambda a, b: float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))
N = 2 * int(meta["nt"]) * int(meta["m"])
rng = np.random.default_rng(1234)
px = rng.standard_normal(N) + 1j * rng.standard_normal(N)
ax = np.asarray(op.apply_A(px)); mx = np.asarray(op.apply_M(px))
print("A sub rel", rel(ax[::16], arr["probe_Ax_sub"]), "norm", np.linalg.norm(ax), float(np.asarray(arr["probe_Ax_norm"])[0]))
print("M sub rel", rel(mx[::16], arr["probe_Mx_sub"]), "norm", np.linalg.norm(mx), float(np.asarray(arr["probe_Mx_norm"])[0]))
x, rep = op.gmres(arr["rhs"][0], rel_tol=meta["gmres_tol"], max_iter=100)
nt, m = meta["nt"], meta["m"]
print("iterations", rep["iterations"], meta["solves"][0]["iterations"], "traces rel", rel(x[: nt * m] + x[nt * m:], arr["ref_traces"][0]))
print("rhs diff vs reference", meta.get("rhs_rel_diff_vs_reference"))
