"""Device-resident polarized interface operator (the uploaded offline state).

``DeviceOperator`` owns one ``pt_handle`` of libpt_b200.so: the entry table
of the polarized "jump" system (trace_system.py:368-472), the sweep
permutation (:353-365) and the kernels (dense Green's blocks or PLR leaves)
uploaded once to HBM.  Its methods are the device versions of the
reference's online operators:

=======================  ===============================================
``apply_A``              ``BlockInterfaceMatrix.matvec`` (:219-226)
``apply_M``              ``preconditioner_apply`` (solver.py:223-228)
``gs_sweep``             ``gs_sweep`` (solver.py:203-220)
``gmres``                ``gmres_solve`` (solver.py:231-295) on the device
=======================  ===============================================

Vectors may be numpy arrays (copied to and from the device) or torch
complex128 CUDA tensors (used in place, stream-ordered on the current
torch stream).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import _native as nat
from .cache import read_case

__all__ = ["DeviceOperator", "load_case_arrays"]

_ENTRY_DT = np.dtype([("row", "<i8"), ("col", "<i8"), ("kernel", "<i8"),
                      ("scale_re", "<f8"), ("scale_im", "<f8"),
                      ("eye_re", "<f8"), ("eye_im", "<f8")])


def _torch():
    import torch
    return torch


def _writable(a):
    """A contiguous array torch.from_numpy can wrap without a warning: read-only
    inputs (memory-mapped case files) are copied first."""
    a = np.ascontiguousarray(a)
    return a if a.flags.writeable else a.copy()


def load_case_arrays(path):
    """(meta, arrays) of a PTC1 case; resolves ``operator_case`` links."""
    path = Path(path)
    meta, arrays = read_case(path)
    link = meta.get("operator_case")
    if link:
        ometa, oarr = read_case(path.with_name(f"{link}.ptc"))
        for k in ("entries", "coefs", "perm", "dense", "leaves", "factors", "kernel_bytes"):
            if k in oarr:
                arrays[k] = oarr[k]
        for k in ("kernel_format", "n_kernels", "kernel_bytes"):
            if k in ometa:
                meta[k] = ometa[k]
    return meta, arrays


class DeviceOperator:
    def __init__(self, *, m, n_block_rows, entries, coefs, perm, dense=None, leaves=None,
                 factors=None, device=None):
        torch = _torch()
        lib = nat.lib()
        if device == "host":  # plan-only handle: host tables, pt_plan_stats (no GPU)
            self.device = nat.PT_DEVICE_HOST
        else:
            if not torch.cuda.is_available():
                raise RuntimeError("DeviceOperator needs a CUDA device (no CPU fallback)")
            self.device = torch.cuda.current_device() if device is None else int(device)
        self.m = int(m)
        self.n_block_rows = int(n_block_rows)
        self.N = self.m * self.n_block_rows
        self.nt = self.n_block_rows // 2
        entries = np.asarray(entries, dtype=np.int64).reshape(-1, 3)
        coefs = np.asarray(coefs, dtype=np.complex128).reshape(-1, 2)
        ent = np.zeros(entries.shape[0], dtype=_ENTRY_DT)
        ent["row"], ent["col"], ent["kernel"] = entries[:, 0], entries[:, 1], entries[:, 2]
        ent["scale_re"], ent["scale_im"] = coefs[:, 0].real, coefs[:, 0].imag
        ent["eye_re"], ent["eye_im"] = coefs[:, 1].real, coefs[:, 1].imag
        self.perm = np.ascontiguousarray(np.asarray(perm, dtype=np.int64))
        self.entries = entries
        self.coefs = coefs
        lay = nat.Layout()
        lay.m = self.m
        lay.n_block_rows = self.n_block_rows
        if dense is not None:
            dense = np.ascontiguousarray(dense, dtype=np.complex128)
            lay.kernel_format = nat.PT_KERNEL_DENSE
            lay.n_kernels = dense.shape[0]
            self.kernel_format = "dense"
            dptr, lptr, nleaf, fptr, nfac = dense.ctypes.data, None, 0, None, 0
        else:
            leaves = np.ascontiguousarray(np.asarray(leaves, dtype=np.int64).reshape(-1, 8))
            factors = np.ascontiguousarray(factors, dtype=np.complex128)
            lay.kernel_format = nat.PT_KERNEL_PLR
            kmax = int(entries[:, 2].max()) + 1 if entries.size else 0
            lay.n_kernels = max(kmax, int(leaves[:, 0].max()) + 1 if leaves.size else 0)
            self.kernel_format = "plr"
            dptr = None
            lptr = leaves.ctypes.data_as(C.POINTER(nat.Leaf))
            nleaf = leaves.shape[0]
            fptr = factors.ctypes.data
            nfac = factors.shape[0]
        self.n_kernels = lay.n_kernels
        h = C.c_void_p()
        rc = lib.pt_create(C.byref(lay), ent.ctypes.data_as(C.POINTER(nat.Entry)), ent.shape[0],
                           self.perm.ctypes.data_as(C.POINTER(C.c_int64)), dptr, lptr, nleaf,
                           fptr, nfac, self.device, C.byref(h))
        nat.check(rc, "pt_create")
        self._h = h

    # ------------------------------------------------------------------
    @classmethod
    def from_case(cls, path, device=None):
        meta, arr = load_case_arrays(path)
        op = cls.from_arrays(meta, arr, device=device)
        op.meta = meta
        return op

    @classmethod
    def from_arrays(cls, meta, arr, device=None):
        n_block_rows = int(meta.get("n_block_rows", 2 * meta.get("nt", 0)))
        kw = dict(m=meta["m"], n_block_rows=n_block_rows, entries=arr["entries"],
                  coefs=arr["coefs"], perm=arr["perm"], device=device)
        if "dense" in arr:
            kw["dense"] = arr["dense"]
        else:
            kw["leaves"], kw["factors"] = arr["leaves"], arr["factors"]
        return cls(**kw)

    @classmethod
    def from_reference(cls, pol, perm, device=None):
        """Upload a reference ``state.pol`` / ``state.perm`` pair."""
        from .capture import capture_operator
        meta, arr = capture_operator(pol, perm)
        return cls.from_arrays(meta, arr, device=device)

    PLAN_STATS = ("tasks", "t_plr", "y_plr", "y_dense", "pieces", "items", "counters",
                  "algo_bytes", "staged_bytes", "max_terms", "max_pieces", "max_items")

    def plan_stats(self, kind="AM", n_it=2):
        """Host-side plan of one program (no launch): task / piece / byte counts."""
        kinds = {"A": 0, "M": 1, "AM": 2, "S": 3}
        st = (C.c_int64 * len(self.PLAN_STATS))()
        nat.check(nat.lib().pt_plan_stats(self._h, kinds[kind], int(n_it), st), "pt_plan_stats")
        return dict(zip(self.PLAN_STATS, (int(v) for v in st)))

    def close(self):
        if getattr(self, "_h", None):
            nat.lib().pt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    def stream(self):
        return C.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _dev_vec(self, x, name="vector"):
        """(tensor on device, was_numpy)."""
        torch = _torch()
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.complex128 or x.device.type != "cuda" or x.device.index != self.device:
                raise ValueError(f"{name} must be a complex128 tensor on cuda:{self.device}")
            if x.shape != (self.N,):
                raise ValueError(f"polarized vector has length {tuple(x.shape)}, expected {self.N}")
            return x.contiguous(), False
        a = np.asarray(x, dtype=np.complex128)
        if a.shape != (self.N,):
            raise ValueError(f"polarized vector has length {a.shape[0] if a.ndim else a.shape}, "
                             f"expected {self.N}")
        return torch.from_numpy(_writable(a)).to(f"cuda:{self.device}"), True

    def _out(self, out, host):
        torch = _torch()
        if out is None:
            return torch.empty(self.N, dtype=torch.complex128, device=f"cuda:{self.device}")
        if host:
            raise ValueError("out= is only supported for CUDA tensor inputs")
        return out

    @staticmethod
    def _ret(t, host):
        return t.cpu().numpy() if host else t

    def apply_A(self, x, out=None):
        xd, host = self._dev_vec(x)
        y = self._out(out, host)
        nat.check(nat.lib().pt_apply_A(self._h, xd.data_ptr(), y.data_ptr(), self.stream()),
                  "pt_apply_A")
        return self._ret(y, host)

    def apply_M(self, r, n_it=2, out=None):
        rd, host = self._dev_vec(r)
        z = self._out(out, host)
        nat.check(nat.lib().pt_apply_M(self._h, rd.data_ptr(), z.data_ptr(), int(n_it),
                                       self.stream()), "pt_apply_M")
        return self._ret(z, host)

    def apply_AM(self, x, n_it=2, out=None):
        """w = M^-1 (A x) in one fused launch (one GMRES iteration's operator work)."""
        xd, host = self._dev_vec(x)
        w = self._out(out, host)
        nat.check(nat.lib().pt_apply_AM(self._h, xd.data_ptr(), w.data_ptr(), int(n_it),
                                        self.stream()), "pt_apply_AM")
        return self._ret(w, host)

    def gs_sweep(self, rhs, u_in, out=None):
        rd, host = self._dev_vec(rhs, "rhs")
        ud, _ = self._dev_vec(u_in, "u_in")
        z = self._out(out, host)
        nat.check(nat.lib().pt_gs_sweep(self._h, rd.data_ptr(), ud.data_ptr(), z.data_ptr(),
                                        self.stream()), "pt_gs_sweep")
        return self._ret(z, host)

    def gmres(self, b, rel_tol=1e-7, max_iter=100, n_it=2, out=None):
        """Device GMRES; returns (x, report dict).  The whole solve is one CUDA
        graph (conditional WHILE node): the host synchronises once per solve
        (PT_GRAPH=0: host-driven, one sync per batch of iterations)."""
        bd, host = self._dev_vec(b, "b")
        x = self._out(out, host)
        cfg = nat.GmresConfigC(float(rel_tol), int(max_iter), int(n_it))
        hist = (C.c_double * int(max_iter))()
        rep = nat.Report()
        rep.residual_history = C.cast(hist, C.POINTER(C.c_double))
        rc = nat.lib().pt_gmres(self._h, bd.data_ptr(), x.data_ptr(), C.byref(cfg), C.byref(rep),
                                self.stream())
        nat.check(rc, "pt_gmres")
        return self._ret(x, host), _report_dict(rep, hist)

    def gmres_host(self, b_host, x_host, rel_tol=1e-7, max_iter=100, n_it=2):
        """GMRES from HOST buffers (pinned torch tensors or numpy): H2D, solve, D2H."""
        cfg = nat.GmresConfigC(float(rel_tol), int(max_iter), int(n_it))
        hist = (C.c_double * int(max_iter))()
        rep = nat.Report()
        rep.residual_history = C.cast(hist, C.POINTER(C.c_double))
        bp = b_host.data_ptr() if hasattr(b_host, "data_ptr") else b_host.ctypes.data
        xp = x_host.data_ptr() if hasattr(x_host, "data_ptr") else x_host.ctypes.data
        rc = nat.lib().pt_gmres_host(self._h, bp, xp, C.byref(cfg), C.byref(rep), self.stream())
        nat.check(rc, "pt_gmres_host")
        return _report_dict(rep, hist)

    # ---- multi-RHS (one row per source; the reference loops sources,
    # cli.py:380-409) ------------------------------------------------------
    def _dev_block(self, X, name="sources"):
        """(nrhs x N complex128 tensor on the device, was_numpy)."""
        torch = _torch()
        if isinstance(X, torch.Tensor):
            if X.dtype != torch.complex128 or X.device.type != "cuda" or X.device.index != self.device:
                raise ValueError(f"{name} must be a complex128 tensor on cuda:{self.device}")
            if X.ndim != 2 or X.shape[1] != self.N:
                raise ValueError(f"{name} must have shape (nrhs, {self.N}), got {tuple(X.shape)}")
            return X.contiguous(), False
        a = np.asarray(X, dtype=np.complex128)
        if a.ndim != 2 or a.shape[1] != self.N:
            raise ValueError(f"{name} must have shape (nrhs, {self.N}), got {a.shape}")
        return torch.from_numpy(_writable(a)).to(f"cuda:{self.device}"), True

    def apply_A_batch(self, X):
        """Y[s] = pol @ X[s] for every source row s (dense operators)."""
        Xd, host = self._dev_block(X)
        Y = _torch().empty_like(Xd)
        nat.check(nat.lib().pt_apply_A_batch(self._h, Xd.data_ptr(), Y.data_ptr(), int(Xd.shape[0]),
                                             self.stream()), "pt_apply_A_batch")
        return self._ret(Y, host)

    def apply_M_batch(self, R, n_it=2):
        """Z[s] = preconditioner_apply(R[s]) for every source row s (dense operators)."""
        Rd, host = self._dev_block(R)
        Z = _torch().empty_like(Rd)
        nat.check(nat.lib().pt_apply_M_batch(self._h, Rd.data_ptr(), Z.data_ptr(), int(Rd.shape[0]),
                                             int(n_it), self.stream()), "pt_apply_M_batch")
        return self._ret(Z, host)

    @staticmethod
    def _reports(nrhs, max_iter):
        hists = [(C.c_double * int(max_iter))() for _ in range(nrhs)]
        reps = (nat.Report * max(nrhs, 1))()
        for i in range(nrhs):
            reps[i].residual_history = C.cast(hists[i], C.POINTER(C.c_double))
        return reps, hists

    def gmres_batch(self, B, rel_tol=1e-7, max_iter=100, n_it=2):
        """Independent GMRES solves of every source row of B: (X, [report, ...]).
        Dense operators run the sources in lockstep batches of 64."""
        Bd, host = self._dev_block(B, "b")
        X = _torch().empty_like(Bd)
        nrhs = int(Bd.shape[0])
        cfg = nat.GmresConfigC(float(rel_tol), int(max_iter), int(n_it))
        reps, hists = self._reports(nrhs, max_iter)
        rc = nat.lib().pt_gmres_batch(self._h, Bd.data_ptr(), X.data_ptr(), nrhs, C.byref(cfg), reps,
                                      self.stream())
        nat.check(rc, "pt_gmres_batch")
        return self._ret(X, host), [_report_dict(reps[i], hists[i]) for i in range(nrhs)]

    def gmres_batch_host(self, B_host, X_host, rel_tol=1e-7, max_iter=100, n_it=2):
        """Batched GMRES from HOST buffers (nrhs x N, pinned torch or numpy)."""
        nrhs = int(B_host.shape[0])
        cfg = nat.GmresConfigC(float(rel_tol), int(max_iter), int(n_it))
        reps, hists = self._reports(nrhs, max_iter)
        bp = B_host.data_ptr() if hasattr(B_host, "data_ptr") else B_host.ctypes.data
        xp = X_host.data_ptr() if hasattr(X_host, "data_ptr") else X_host.ctypes.data
        rc = nat.lib().pt_gmres_batch_host(self._h, bp, xp, nrhs, C.byref(cfg), reps, self.stream())
        nat.check(rc, "pt_gmres_batch_host")
        return [_report_dict(reps[i], hists[i]) for i in range(nrhs)]

    def exec_timing(self, enable=True):
        """Bracket every executor launch with CUDA events (resets the stats)."""
        nat.check(nat.lib().pt_exec_timing(self._h, 1 if enable else 0), "pt_exec_timing")

    def exec_stats(self):
        """(device ms summed over timed launches, launches, algorithmic bytes)."""
        ms, n, b = C.c_double(), C.c_int64(), C.c_int64()
        nat.check(nat.lib().pt_exec_stats(self._h, C.byref(ms), C.byref(n), C.byref(b)),
                  "pt_exec_stats")
        return float(ms.value), int(n.value), int(b.value)

    def exec_info(self):
        """{'grid': CTAs, 'smem': bytes per CTA, 'half_elems': staging half (complex)}."""
        g, sm, hf = C.c_int32(), C.c_int64(), C.c_int64()
        nat.check(nat.lib().pt_exec_info(self._h, C.byref(g), C.byref(sm), C.byref(hf)), "info")
        return {"grid": int(g.value), "smem": int(sm.value), "half_elems": int(hf.value)}

    def bytes_apply_A(self):
        return int(nat.lib().pt_bytes_apply_A(self._h))

    def bytes_apply_M(self, n_it=2):
        return int(nat.lib().pt_bytes_apply_M(self._h, int(n_it)))


def _report_dict(rep, hist):
    k = int(rep.iterations)
    return {
        "iterations": k,
        "flag": nat.FLAGS.get(int(rep.flag), "unknown"),
        "converged": bool(rep.converged),
        "true_residual": float(rep.true_residual),
        "beta": float(rep.beta),
        "residual_history": [float(hist[i]) for i in range(k)],
    }
