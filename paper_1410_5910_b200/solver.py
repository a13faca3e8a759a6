"""Reference-shaped online solver API, routed to the device.

Mirrors the public names of the reference's ``helmsweep.solver`` (the
``__all__`` at solver.py:40-53) so a caller switches by changing the
import.  The online GMRES stage runs through libpt_b200.so on the GPU; the
offline stage and the host online stages (restrict, Newton traces, volume
reconstruction) stay the reference's host code, exactly as the north star
prescribes, and are only reachable where the reference package is
importable.  There is no CPU fallback for the device stage: without the
CUDA library every entry point raises.

================================  =========================================
this module                       reference
================================  =========================================
PreconditionerConfig              solver.py:59-68
GmresConfig                       solver.py:71-80
CompressionConfig                 solver.py:83-93
SolveReport                       solver.py:96-107
OfflineState                      solver.py:110-129 (+ the device handle)
offline_assemble                  solver.py:132-193 (host) + one upload
gs_sweep                          solver.py:203-220
preconditioner_apply              solver.py:223-228
gmres_solve                       solver.py:231-295
solve_online                      solver.py:376-401 (the "gmres" stage)
solve_helmholtz                   solver.py:308-435
================================  =========================================
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .operator import DeviceOperator, load_case_arrays

__all__ = [
    "PreconditionerConfig",
    "GmresConfig",
    "CompressionConfig",
    "SolveReport",
    "OfflineState",
    "offline_assemble",
    "gs_sweep",
    "preconditioner_apply",
    "gmres_solve",
    "solve_online",
    "solve_helmholtz",
]

STAGNATION_WINDOW = 10          # solver.py:55
STAGNATION_IMPROVEMENT = 1e-3   # solver.py:56


@dataclass
class PreconditionerConfig:
    n_it: int = 2
    variant: str = "jump"

    def __post_init__(self):
        if self.n_it < 1:
            raise ValueError("n_it must be at least 1")
        if self.variant not in ("jump", "extrapolation"):
            raise ValueError(f"unknown preconditioner variant {self.variant!r}")


@dataclass
class GmresConfig:
    rel_tol: float = 1e-7
    max_iter: int = 100

    def __post_init__(self):
        if not 0.0 < self.rel_tol < 1.0:
            raise ValueError("rel_tol must lie in (0, 1)")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")


@dataclass
class CompressionConfig:
    """PLR compression switch, forwarded to the reference offline stage."""

    epsilon: float | None = None
    r_max: int | None = None


@dataclass
class SolveReport:
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    flag: str = "converged"
    true_residual: float | None = None
    traces: np.ndarray | None = None
    layer_fields: list | None = None
    u: np.ndarray | None = None
    stage_seconds: dict = field(default_factory=dict)
    oracle_rel_error: float | None = None


# ----------------------------------------------------------------------------
# device views standing in for BlockInterfaceMatrix / SplitD / SplitR


class DevicePolarized:
    """``state.pol``: ``matvec`` is the device A-apply (trace_system.py:219-226)."""

    def __init__(self, op: DeviceOperator):
        self.op = op
        self.m = op.m
        self.n_block_rows = self.n_block_cols = op.n_block_rows

    @property
    def shape(self):
        return (self.op.N, self.op.N)

    def matvec(self, x):
        return self.op.apply_A(x)


@dataclass
class DeviceSplitD:
    op: DeviceOperator


@dataclass
class DeviceSplitR:
    op: DeviceOperator


class DevicePreconditioner:
    """Callable ``r -> preconditioner_apply(config, d, r, perm, r)`` on the device."""

    def __init__(self, op: DeviceOperator, config: PreconditionerConfig):
        self.op = op
        self.config = config

    def __call__(self, residual):
        return self.op.apply_M(residual, n_it=self.config.n_it)


@dataclass
class OfflineState:
    """Device-resident offline state (plus the reference host state if any)."""

    op: DeviceOperator
    variant: str = "jump"
    host_state: object = None
    meta: dict = field(default_factory=dict)
    stage_seconds: dict = field(default_factory=dict)
    # device layer factorizations (Newton traces / reconstruction on the GPU)
    local: object = None

    @property
    def pol(self):
        return DevicePolarized(self.op)

    @property
    def d(self):
        return DeviceSplitD(self.op)

    @property
    def r(self):
        return DeviceSplitR(self.op)

    @property
    def perm(self):
        return self.op.perm

    @property
    def block_size(self) -> int:
        return self.op.m

    @property
    def n_traces(self) -> int:
        return self.op.nt

    def preconditioner(self, config: PreconditionerConfig | None = None):
        return DevicePreconditioner(self.op, config or PreconditionerConfig())

    @classmethod
    def from_case(cls, path, device=None, local=False):
        """A PTC1 operator cache; ``local=True`` also factors the case's layers
        for the device Newton / reconstruction stages (offline/local.py)."""
        meta, arr = load_case_arrays(path)
        op = DeviceOperator.from_arrays(meta, arr, device=device)
        op.meta = meta
        state = cls(op=op, variant=meta.get("variant", "jump"), meta=meta)
        if local:
            from .local import DeviceLocalSolver
            t0 = time.perf_counter()
            state.local = DeviceLocalSolver.from_config(meta["name"], device=device)
            state.stage_seconds["local_factor"] = time.perf_counter() - t0
        return state


def offline_assemble(grid, model, part, omega, *, variant="jump", factor_method="banded",
                     compression=None, profile=None, device=None) -> OfflineState:
    """Reference host offline stage (solver.py:132-193), then one upload."""
    try:
        from helmsweep import solver as ref_solver
    except ImportError as exc:  # pragma: no cover - depends on the host
        raise ImportError("offline_assemble needs the reference package `helmsweep` "
                          "(its offline stage is host code that stays the reference's); "
                          "load a PTC1 operator cache with OfflineState.from_case instead") from exc
    comp = None
    if compression is not None:
        comp = ref_solver.CompressionConfig(epsilon=compression.epsilon, r_max=compression.r_max)
    host = ref_solver.offline_assemble(grid, model, part, omega, variant=variant,
                                       factor_method=factor_method, compression=comp,
                                       profile=profile)
    t0 = time.perf_counter()
    op = DeviceOperator.from_reference(host.pol, host.perm, device=device)
    stages = dict(host.stage_seconds)
    stages["upload"] = time.perf_counter() - t0
    return OfflineState(op=op, variant=variant, host_state=host, stage_seconds=stages)


def _device_op(d, r, perm) -> DeviceOperator:
    if not isinstance(d, DeviceSplitD) or not isinstance(r, DeviceSplitR) or d.op is not r.op:
        raise TypeError("device sweeps need state.d / state.r of one device OfflineState")
    if not np.array_equal(np.asarray(perm), d.op.perm):
        raise ValueError("permutation does not match the uploaded sweep order")
    return d.op


def gs_sweep(d, r, perm, rhs, u_in):
    """One stationary step u_next = D^-1 (P rhs - R u_in) on the device."""
    return _device_op(d, r, perm).gs_sweep(rhs, u_in)


def preconditioner_apply(config: PreconditionerConfig, d, r, perm, residual):
    """n_it sweeps from zero on the device; a fixed linear operator."""
    return _device_op(d, r, perm).apply_M(residual, n_it=config.n_it)


# ----------------------------------------------------------------------------
# GMRES


def _fused_target(apply_A, apply_Minv):
    owner = getattr(apply_A, "__self__", None)
    if isinstance(owner, DevicePolarized) and isinstance(apply_Minv, DevicePreconditioner) \
            and apply_Minv.op is owner.op and getattr(apply_A, "__func__", None) is DevicePolarized.matvec:
        return owner.op, apply_Minv.config.n_it
    return None


def gmres_solve(apply_A, apply_Minv, b, config: GmresConfig):
    """Left-preconditioned GMRES (no restart) with the Arnoldi/Givens work on the GPU.

    With ``state.pol.matvec`` and ``state.preconditioner(...)`` the whole
    iteration runs on the device (libpt_b200 ``pt_gmres``).  Any other
    callables are applied by the caller's code between device Arnoldi steps
    (``pt_gmres_ws_*``); they receive and return numpy arrays when ``b`` is a
    numpy array and CUDA tensors when ``b`` is a CUDA tensor.
    """
    fused = _fused_target(apply_A, apply_Minv)
    if fused is not None:
        op, n_it = fused
        x, rep = op.gmres(b, rel_tol=config.rel_tol, max_iter=config.max_iter, n_it=n_it)
        return x, _to_report(rep)
    return _gmres_callables(apply_A, apply_Minv, b, config)


def _to_report(rep: dict) -> SolveReport:
    out = SolveReport()
    out.iterations = rep["iterations"]
    out.residual_history = list(rep["residual_history"])
    out.converged = rep["converged"]
    out.flag = rep["flag"]
    out.true_residual = rep["true_residual"]
    return out


def _gmres_callables(apply_A, apply_Minv, b, config: GmresConfig):
    import ctypes as C

    import torch

    lib = nat.lib()
    host = not isinstance(b, torch.Tensor)
    if host:
        b_np = np.asarray(b, dtype=np.complex128)
        n = b_np.shape[0]
        dev = torch.cuda.current_device()
        bd = torch.from_numpy(np.ascontiguousarray(b_np)).to(f"cuda:{dev}")
    else:
        bd = b.to(torch.complex128).contiguous()
        dev = bd.device.index
        n = bd.shape[0]

    def call(fn, v_dev):
        if host:
            out = np.asarray(fn(v_dev.cpu().numpy()), dtype=np.complex128)
            return torch.from_numpy(np.ascontiguousarray(out)).to(f"cuda:{dev}")
        return fn(v_dev).to(torch.complex128).contiguous()

    ws = C.c_void_p()
    nat.check(lib.pt_gmres_ws_create(n, config.max_iter, dev, C.byref(ws)), "ws_create")
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    report = SolveReport()
    try:
        def basis(j):
            ptr = lib.pt_gmres_ws_basis(ws, j)
            return _wrap_device(ptr, n, dev)

        mb = call(apply_Minv, bd)
        beta = C.c_double()
        nat.check(lib.pt_gmres_ws_begin(ws, mb.data_ptr(), C.byref(beta), stream), "ws_begin")
        x = torch.zeros(n, dtype=torch.complex128, device=f"cuda:{dev}")
        if beta.value == 0.0:
            report.converged = True
            report.true_residual = 0.0
            return (x.cpu().numpy() if host else x), report
        hist = (C.c_double * config.max_iter)()
        rep = nat.Report()
        rep.residual_history = C.cast(hist, C.POINTER(C.c_double))
        stop = C.c_int32(0)
        for j in range(config.max_iter):
            w = call(apply_Minv, call(apply_A, basis(j)))
            basis(j + 1).copy_(w)
            torch.cuda.current_stream(dev).synchronize()
            rc = lib.pt_gmres_ws_step(ws, j, config.rel_tol, config.max_iter, C.byref(rep),
                                      C.byref(stop), stream)
            nat.check(rc, "ws_step")
            if stop.value:
                break
        k = int(rep.iterations)
        nat.check(lib.pt_gmres_ws_finish(ws, k, x.data_ptr(), stream), "ws_finish")
        report.iterations = k
        report.residual_history = [float(hist[i]) for i in range(k)]
        report.converged = bool(rep.converged)
        report.flag = nat.FLAGS[int(rep.flag)]
        ax = call(apply_A, x)
        true_res = torch.linalg.vector_norm(bd - ax).item()
        scale = torch.linalg.vector_norm(bd).item()
        report.true_residual = float(true_res / scale) if scale > 0 else float(true_res)
        return (x.cpu().numpy() if host else x), report
    finally:
        torch.cuda.current_stream(dev).synchronize()
        lib.pt_gmres_ws_destroy(ws)


def _wrap_device(ptr, n, dev):
    """A torch view of n complex128 at a raw device pointer (library-owned)."""
    import torch

    class _Holder:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {
                "shape": (n,), "typestr": "<c16", "data": (p, False), "version": 3,
                "strides": None,
            }

    return torch.as_tensor(_Holder(ptr, n), device=f"cuda:{dev}")


# ----------------------------------------------------------------------------
# online pipeline


def solve_online(state: OfflineState, rhs, precond: PreconditionerConfig | None = None,
                 gmres: GmresConfig | None = None) -> tuple:
    """The "gmres" stage of solve_helmholtz (solver.py:376-401) on the device.

    Returns (x, report) with report.traces = x_down + x_up stacked
    (TraceVector.from_flat, trace_system.py:83-88).
    """
    precond = precond or PreconditionerConfig()
    gmres = gmres or GmresConfig()
    if state.variant != precond.variant:
        raise ValueError(f"offline state was assembled for variant {state.variant!r}, "
                         f"preconditioner wants {precond.variant!r}")
    report = SolveReport()
    nt, m = state.n_traces, state.block_size
    rhs_np = None if hasattr(rhs, "data_ptr") else np.asarray(rhs, dtype=np.complex128)
    is_zero = bool((rhs_np == 0).all()) if rhs_np is not None else not bool(rhs.abs().max() > 0)
    t0 = time.perf_counter()
    if is_zero:
        x = np.zeros(2 * nt * m, dtype=np.complex128) if rhs_np is not None else rhs * 0
        report.converged = True
    else:
        x, inner = gmres_solve(state.pol.matvec, state.preconditioner(precond), rhs, gmres)
        report.iterations = inner.iterations
        report.residual_history = inner.residual_history
        report.converged = inner.converged
        report.flag = inner.flag
        report.true_residual = inner.true_residual
    report.stage_seconds["gmres"] = time.perf_counter() - t0
    xn = x if isinstance(x, np.ndarray) else x.cpu().numpy()
    report.traces = xn[: nt * m] + xn[nt * m:]
    return x, report


def _solve_helmholtz_device(state, f, precond, gmres, report, oracle):
    """Every online stage on the device: restrict + newton + rhs
    (pt_local_newton), gmres (pt_gmres), reconstruct (pt_local_reconstruct).
    The host copies f in and u out; one synchronisation per stage."""
    import torch
    loc = state.local

    def stage(name, fn):
        t0 = time.perf_counter()
        try:
            out = fn()
            torch.cuda.synchronize(loc.device)
        except Exception as exc:
            raise RuntimeError(f"stage {name!r} failed: {exc}") from exc
        report.stage_seconds[name] = time.perf_counter() - t0
        return out

    f_dev = stage("restrict", lambda: loc._dev(f, (loc.nz_ext, loc.nxe), "f")[0])
    rhs = stage("rhs", lambda: loc.rhs(f_dev, state.variant))
    x, inner = stage("gmres", lambda: solve_online(state, rhs, precond, gmres))
    for k in ("iterations", "residual_history", "converged", "flag", "true_residual"):
        setattr(report, k, getattr(inner, k))
    report.traces = inner.traces
    x_dev = x if hasattr(x, "data_ptr") else torch.from_numpy(np.array(x, dtype=np.complex128)).to(f_dev.device)
    u = stage("reconstruct", lambda: loc.reconstruct(f_dev, x_dev))
    report.u = u.cpu().numpy()
    n_c = loc.geo["n_c"]
    report.layer_fields = [report.u[n_c[i]:n_c[i + 1]] for i in range(len(n_c) - 1)]
    if oracle is not None:
        scale = np.linalg.norm(oracle)
        err = np.linalg.norm(report.u - oracle)
        report.oracle_rel_error = float(err / scale) if scale > 0 else float(err)
    return report


def solve_helmholtz(model, grid, part, f, *, omega=None, state: OfflineState | None = None,
                    precond=None, gmres=None, factor_method="banded", compression=None,
                    oracle=None) -> SolveReport:
    """solve_helmholtz (solver.py:308-435) with the GMRES stage on the device.

    With ``state.local`` (``OfflineState.from_case(..., local=True)``) every
    online stage runs on the device and model/grid/part are not needed; else
    restrict / newton / rhs / reconstruct are the reference's host stages
    (they need ``state.host_state``, i.e. an OfflineState from
    :func:`offline_assemble`).
    """
    precond = precond or PreconditionerConfig()
    gmres = gmres or GmresConfig()
    report = SolveReport()
    if state is None:
        if omega is None:
            raise ValueError("omega is required when no offline state is given")
        t0 = time.perf_counter()
        try:
            state = offline_assemble(grid, model, part, omega, variant=precond.variant,
                                     factor_method=factor_method, compression=compression)
        except Exception as exc:
            raise RuntimeError(f"stage 'offline' failed: {exc}") from exc
        report.stage_seconds["offline"] = time.perf_counter() - t0
    elif state.variant != precond.variant:
        raise ValueError(f"offline state was assembled for variant {state.variant!r}, "
                         f"preconditioner wants {precond.variant!r}")
    if state.local is not None:
        return _solve_helmholtz_device(state, f, precond, gmres, report, oracle)
    host = state.host_state
    if host is None:
        raise ValueError("solve_helmholtz needs layer factorizations: an OfflineState built by "
                         "offline_assemble, or OfflineState.from_case(..., local=True)")

    from helmsweep.local_solver import newton_trace, reconstruct_volume
    from helmsweep.partition import restrict_source
    from helmsweep.trace_system import TraceVector, polarized_rhs

    def stage(name, fn):
        t0 = time.perf_counter()
        try:
            out = fn()
        except Exception as exc:
            raise RuntimeError(f"stage {name!r} failed: {exc}") from exc
        report.stage_seconds[name] = time.perf_counter() - t0
        return out

    n_pml = grid.n_pml
    f_locals = stage("restrict", lambda: [restrict_source(f, part, ell, n_pml)
                                          for ell in range(1, part.L + 1)])
    newtons = stage("newton", lambda: [newton_trace(host.facts[ell - 1], f_locals[ell - 1],
                                                    part.thickness(ell), n_pml)
                                       for ell in range(1, part.L + 1)])
    rhs = stage("rhs", lambda: polarized_rhs(newtons, part, state.variant))
    x, inner = stage("gmres", lambda: solve_online(state, rhs, precond, gmres))
    for k in ("iterations", "residual_history", "converged", "flag", "true_residual"):
        setattr(report, k, getattr(inner, k))
    nt, m = state.n_traces, state.block_size
    traces = TraceVector.from_flat(inner.traces, m)
    report.traces = traces.stack()

    def rebuild():
        fields = []
        for ell in range(1, part.L + 1):
            top, bot = 2 * (ell - 2), 2 * (ell - 1)
            fields.append(reconstruct_volume(
                host.facts[ell - 1], f_locals[ell - 1],
                traces.blocks[top] if ell >= 2 else None,
                traces.blocks[top + 1] if ell >= 2 else None,
                traces.blocks[bot] if ell <= part.L - 1 else None,
                traces.blocks[bot + 1] if ell <= part.L - 1 else None,
                part.thickness(ell), n_pml, grid.h))
        return fields

    report.layer_fields = stage("reconstruct", rebuild)
    report.u = np.concatenate(report.layer_fields, axis=0)
    if oracle is not None:
        scale = np.linalg.norm(oracle)
        err = np.linalg.norm(report.u - oracle)
        report.oracle_rel_error = float(err / scale) if scale > 0 else float(err)
    return report
