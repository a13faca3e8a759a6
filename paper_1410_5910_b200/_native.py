"""ctypes binding of the C ABI in ``include/pt_b200.h`` (libpt_b200.so).

This is exactly the binding a maintainer would add to the reference to
route its online stage to the device.  The library is
required: there is no CPU fallback, and importing the operator classes
without it raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PT_B200_LIB", _HERE / "libpt_b200.so"))
# PT_LIBRARY=check loads the checked build (libpt_b200_check.so: invariant
# asserts and spin-loop watchdogs in the executor; csrc/Makefile `check`)
if os.environ.get("PT_LIBRARY") == "check":
    LIB_PATH = LIB_PATH.with_name("libpt_b200_check.so")

PT_OK, PT_EINVAL, PT_ECUDA, PT_ENONFINITE = 0, -1, -2, -3
PT_KERNEL_DENSE, PT_KERNEL_PLR = 0, 1
PT_DEVICE_HOST = -1
FLAGS = {0: "converged", 1: "breakdown", 2: "stagnation", 3: "maxiter"}


class Layout(C.Structure):
    _fields_ = [("m", C.c_int64), ("n_block_rows", C.c_int64),
                ("kernel_format", C.c_int32), ("n_kernels", C.c_int32)]


class Entry(C.Structure):
    _fields_ = [("row", C.c_int64), ("col", C.c_int64), ("kernel", C.c_int64),
                ("scale_re", C.c_double), ("scale_im", C.c_double),
                ("eye_re", C.c_double), ("eye_im", C.c_double)]


class Leaf(C.Structure):
    _fields_ = [("kernel", C.c_int64), ("row_off", C.c_int64), ("col_off", C.c_int64),
                ("rows", C.c_int64), ("cols", C.c_int64), ("rank", C.c_int64),
                ("u_off", C.c_int64), ("vt_off", C.c_int64)]


class GmresConfigC(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int32), ("n_it", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("flag", C.c_int32), ("converged", C.c_int32),
                ("nonfinite", C.c_int32), ("true_residual", C.c_double), ("beta", C.c_double),
                ("residual_history", C.POINTER(C.c_double))]


class LocalLayer(C.Structure):
    _fields_ = [("dim", C.c_int64), ("nze", C.c_int64), ("nxe", C.c_int64),
                ("n_layer", C.c_int64), ("n_pml", C.c_int64),
                ("l_ptr", C.c_void_p), ("l_col", C.c_void_p), ("l_val", C.c_void_p),
                ("u_ptr", C.c_void_p), ("u_col", C.c_void_p), ("u_val", C.c_void_p),
                ("q_in", C.c_void_p), ("q_out", C.c_void_p),
                ("n_blocks", C.c_int64), ("block_ptr", C.c_void_p)]


_VP = C.c_void_p
_SIGS = {
    "pt_create": (C.c_int, [C.POINTER(Layout), C.POINTER(Entry), C.c_int64, C.POINTER(C.c_int64),
                            _VP, C.POINTER(Leaf), C.c_int64, _VP, C.c_int64, C.c_int,
                            C.POINTER(_VP)]),
    "pt_destroy": (C.c_int, [_VP]),
    "pt_apply_A": (C.c_int, [_VP, _VP, _VP, _VP]),
    "pt_apply_M": (C.c_int, [_VP, _VP, _VP, C.c_int32, _VP]),
    "pt_gs_sweep": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "pt_apply_AM": (C.c_int, [_VP, _VP, _VP, C.c_int32, _VP]),
    "pt_gmres": (C.c_int, [_VP, _VP, _VP, C.POINTER(GmresConfigC), C.POINTER(Report), _VP]),
    "pt_gmres_host": (C.c_int, [_VP, _VP, _VP, C.POINTER(GmresConfigC), C.POINTER(Report), _VP]),
    "pt_gmres_batch": (C.c_int, [_VP, _VP, _VP, C.c_int32, C.POINTER(GmresConfigC),
                                 C.POINTER(Report), _VP]),
    "pt_gmres_batch_host": (C.c_int, [_VP, _VP, _VP, C.c_int32, C.POINTER(GmresConfigC),
                                      C.POINTER(Report), _VP]),
    "pt_apply_A_batch": (C.c_int, [_VP, _VP, _VP, C.c_int32, _VP]),
    "pt_apply_M_batch": (C.c_int, [_VP, _VP, _VP, C.c_int32, C.c_int32, _VP]),
    "pt_gmres_ws_create": (C.c_int, [C.c_int64, C.c_int32, C.c_int, C.POINTER(_VP)]),
    "pt_gmres_ws_destroy": (C.c_int, [_VP]),
    "pt_gmres_ws_basis": (_VP, [_VP, C.c_int32]),
    "pt_gmres_ws_begin": (C.c_int, [_VP, _VP, C.POINTER(C.c_double), _VP]),
    "pt_gmres_ws_step": (C.c_int, [_VP, C.c_int32, C.c_double, C.c_int32, C.POINTER(Report),
                                   C.POINTER(C.c_int32), _VP]),
    "pt_gmres_ws_finish": (C.c_int, [_VP, C.c_int32, _VP, _VP]),
    "pt_exec_timing": (C.c_int, [_VP, C.c_int32]),
    "pt_exec_stats": (C.c_int, [_VP, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64)]),
    "pt_trace_program": (C.c_int, [_VP, C.c_int32, C.c_int32, _VP, _VP, C.POINTER(C.c_int64),
                                   C.c_int64, C.POINTER(C.c_int64)]),
    "pt_plan_stats": (C.c_int, [_VP, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "pt_plan_tasks": (C.c_int, [_VP, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int64,
                               C.POINTER(C.c_int64)]),
    "pt_exec_info": (C.c_int, [_VP, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)]),
    "pt_local_create": (C.c_int, [C.POINTER(LocalLayer), C.c_int32, C.c_int, C.POINTER(_VP)]),
    "pt_local_destroy": (C.c_int, [_VP]),
    "pt_local_info": (C.c_int, [_VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "pt_local_solve": (C.c_int, [_VP, _VP, _VP, _VP]),
    "pt_local_newton": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int32, _VP]),
    "pt_local_reconstruct": (C.c_int, [_VP, _VP, _VP, C.c_double, _VP, _VP]),
    "pt_local_last_error": (C.c_char_p, []),
    "pt_last_error": (C.c_char_p, []),
    "pt_abi_version": (C.c_int32, []),
    "pt_launch_count": (C.c_int64, []),
    "pt_checked_build": (C.c_int32, []),
    "pt_bytes_apply_A": (C.c_int64, [_VP]),
    "pt_bytes_apply_M": (C.c_int64, [_VP, C.c_int32]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libpt_b200.so once; raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_1410_5910_b200/csrc` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.pt_abi_version() != 1:
            raise ImportError("libpt_b200.so ABI version mismatch")
        _lib = handle
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types."""
    if rc == PT_OK:
        return
    msg = lib().pt_last_error().decode(errors="replace")
    if rc == PT_EINVAL:
        raise ValueError(msg)
    if rc == PT_ENONFINITE:
        raise RuntimeError(msg)
    raise RuntimeError(f"CUDA failure{(' in ' + what) if what else ''}: {msg}")
