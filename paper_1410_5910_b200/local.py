"""Device local solves: Newton traces, polarized right-hand side and volume
reconstruction of every layer at once.

Mirrors the reference's host stages of ``solve_helmholtz`` (solver.py:355-426):
``newton_trace`` (local_solver.py:138-144) + ``polarized_rhs``
(trace_system.py:475-484) and ``reconstruct_volume`` (local_solver.py:147-176),
through the C ABI ``pt_local_*`` of ``include/pt_b200.h``.  The layer
factorizations come from the host offline stage (``offline/local.py``).
There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .operator import _writable

__all__ = ["DeviceLocalSolver"]


def _torch():
    import torch
    return torch


class DeviceLocalSolver:
    def __init__(self, factors, geometry, device=None):
        torch = _torch()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.geo = dict(geometry)
        self.nxe = int(self.geo["nxe"])
        self.L = len(factors)
        self.nz = int(sum(f["n_layer"] for f in factors))
        self.nz_ext = self.nz + 2 * int(self.geo["n_pml"])
        self.N = 2 * (2 * self.L - 2) * self.nxe
        keep = []  # host arrays must outlive pt_local_create
        arr = (nat.LocalLayer * self.L)()
        for i, f in enumerate(factors):
            Lm, Um = f["L"], f["U"]
            parts = {
                "l_ptr": np.ascontiguousarray(Lm.indptr, dtype=np.int64),
                "l_col": np.ascontiguousarray(Lm.indices, dtype=np.int32),
                "l_val": np.ascontiguousarray(Lm.data, dtype=np.complex128),
                "u_ptr": np.ascontiguousarray(Um.indptr, dtype=np.int64),
                "u_col": np.ascontiguousarray(Um.indices, dtype=np.int32),
                "u_val": np.ascontiguousarray(Um.data, dtype=np.complex128),
                "q_in": np.ascontiguousarray(f["q_in"], dtype=np.int64),
                "q_out": np.ascontiguousarray(f["q_out"], dtype=np.int64),
            }
            bp = f.get("block_ptr")
            if bp is not None:
                parts["block_ptr"] = np.ascontiguousarray(bp, dtype=np.int64)
            keep.append(parts)
            a = arr[i]
            a.dim = f["nze"] * f["nxe"]
            a.nze, a.nxe, a.n_layer, a.n_pml = f["nze"], f["nxe"], f["n_layer"], f["n_pml"]
            for k, v in parts.items():
                setattr(a, k, v.ctypes.data)
            a.n_blocks = 0 if bp is None else len(bp) - 1
        h = C.c_void_p()
        rc = nat.lib().pt_local_create(arr, self.L, self.device, C.byref(h))
        if rc != 0:
            raise (ValueError if rc == nat.PT_EINVAL else RuntimeError)(
                nat.lib().pt_local_last_error().decode(errors="replace"))
        self._h = h
        rows, nnz, ll, ul = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
        nat.lib().pt_local_info(self._h, C.byref(rows), C.byref(nnz), C.byref(ll), C.byref(ul))
        self.info = {"rows": rows.value, "factor_nnz": nnz.value, "l_levels": ll.value,
                     "u_levels": ul.value,
                     "blocked": all(f.get("block_ptr") is not None for f in factors)}

    @classmethod
    def from_config(cls, name, device=None, workers=None):
        from .offline.local import build_local
        facs, geo = build_local(name, workers=workers)
        return cls(facs, geo, device=device)

    def close(self):
        if getattr(self, "_h", None):
            nat.lib().pt_local_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        return C.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _check(self, rc, what):
        if rc != 0:
            msg = nat.lib().pt_local_last_error().decode(errors="replace")
            raise (ValueError if rc == nat.PT_EINVAL else RuntimeError)(f"{what}: {msg}")

    def _dev(self, a, shape, name):
        torch = _torch()
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.complex128 or a.device.type != "cuda" or tuple(a.shape) != shape:
                raise ValueError(f"{name} must be a complex128 CUDA tensor of shape {shape}")
            return a.contiguous(), False
        a = np.asarray(a, dtype=np.complex128)
        if a.shape != shape:
            raise ValueError(f"{name} has shape {a.shape}, expected {shape}")
        return torch.from_numpy(_writable(a)).to(f"cuda:{self.device}"), True

    def solve(self, b):
        """x_l = H_l^-1 b_l for every layer (layers concatenated, natural order)."""
        torch = _torch()
        bd, host = self._dev(b, (self.info["rows"],), "b")
        x = torch.empty_like(bd)
        self._check(nat.lib().pt_local_solve(self._h, bd.data_ptr(), x.data_ptr(), self._stream()),
                    "pt_local_solve")
        return x.cpu().numpy() if host else x

    def newton(self, f):
        """Newton traces (L, 4, nxe) at local depths 0, 1, n, n+1 (newton_trace)."""
        torch = _torch()
        fd, host = self._dev(f, (self.nz_ext, self.nxe), "f")
        tr = torch.empty((self.L, 4, self.nxe), dtype=torch.complex128, device=fd.device)
        self._check(nat.lib().pt_local_newton(self._h, fd.data_ptr(), tr.data_ptr(), None, 1,
                                              self._stream()), "pt_local_newton")
        return tr.cpu().numpy() if host else tr

    def rhs(self, f, variant="jump"):
        """The polarized right-hand side of source f (newton + polarized_rhs)."""
        torch = _torch()
        if variant not in ("jump", "extrapolation"):
            raise ValueError(f"unknown polarized variant {variant!r}")
        fd, host = self._dev(f, (self.nz_ext, self.nxe), "f")
        out = torch.empty(self.N, dtype=torch.complex128, device=fd.device)
        self._check(nat.lib().pt_local_newton(self._h, fd.data_ptr(), None, out.data_ptr(),
                                              1 if variant == "jump" else 0, self._stream()),
                    "pt_local_newton")
        return out.cpu().numpy() if host else out

    def reconstruct(self, f, x, h=None):
        """Volume u (nz, nxe) from the GMRES solution x (traces x_down + x_up)."""
        torch = _torch()
        fd, host = self._dev(f, (self.nz_ext, self.nxe), "f")
        xd, _ = self._dev(x, (self.N,), "x")
        u = torch.empty((self.nz, self.nxe), dtype=torch.complex128, device=fd.device)
        hh = float(self.geo["h"] if h is None else h)
        self._check(nat.lib().pt_local_reconstruct(self._h, fd.data_ptr(), xd.data_ptr(), hh,
                                                   u.data_ptr(), self._stream()),
                    "pt_local_reconstruct")
        return u.cpu().numpy() if host else u
