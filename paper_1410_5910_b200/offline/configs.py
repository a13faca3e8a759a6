"""BASELINE configurations c1..c5 as seeded synthetic media.

No public dataset is involved: BASELINE.json's configs are themselves
synthetic descriptions; the seeds, draw orders and omega rules below are the
ones SURVEY.md §8(d) fixes (its c_min / c_max / omega values are reproduced
exactly, see tests/test_offline.py).  Geometry follows the reference's own
conventions: h = 1/(nx+1) (cli.py:233), unit-width domain, media given on the
interior and edge-extended into the PML (grid.py:144-149), point sources are
discrete deltas of amplitude 1/h^2 at the nearest interior node
(cli.py:269-274), layers split equally with the remainder to the front
(partition.py:68-84).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Geometry", "CaseConfig", "config", "CASES", "FIXTURES"]


@dataclass(frozen=True)
class Geometry:
    nx: int
    nz: int
    n_pml: int

    @property
    def h(self) -> float:
        return 1.0 / (self.nx + 1)

    @property
    def nx_ext(self) -> int:
        return self.nx + 2 * self.n_pml

    @property
    def nz_ext(self) -> int:
        return self.nz + 2 * self.n_pml

    @property
    def Lx(self) -> float:
        return (self.nx + 1) * self.h

    @property
    def Lz(self) -> float:
        return (self.nz + 1) * self.h

    def x_coords(self):
        return np.arange(-self.n_pml + 1, self.nx + self.n_pml + 1) * self.h

    def z_coords(self):
        return np.arange(-self.n_pml + 1, self.nz + self.n_pml + 1) * self.h

    def interior_xz(self):
        x = self.x_coords()[self.n_pml:self.n_pml + self.nx]
        z = self.z_coords()[self.n_pml:self.n_pml + self.nz]
        return np.meshgrid(x, z)


@dataclass
class CaseConfig:
    name: str
    geo: Geometry
    c: np.ndarray            # interior velocity (nz, nx)
    L: int
    omega: float
    sources: list            # [(label, f on the extended grid)]
    compression: tuple | None  # (epsilon, r_max) or None for dense kernels
    tol: float
    note: str
    extra: dict = field(default_factory=dict)
    variant: str = "jump"    # polarized variant (trace_system.py:368-472)


# ---- media -------------------------------------------------------------------


def medium_homogeneous(g, c0=1.0):
    return np.full((g.nz, g.nx), float(c0))


def medium_gradient(g):
    X, Z = g.interior_xz()
    return 1.0 + 0.1 * X + 0.1 * Z


def medium_bumps(g, seed=2, count=12):
    """c2: 1.5 + sum of seeded Gaussian bumps, clipped to [1.5, 4.5]."""
    X, Z = g.interior_xz()
    rng = np.random.default_rng(seed)
    c = np.full_like(X, 1.5)
    for _ in range(count):
        xk = rng.uniform(0.0, 1.0, size=2)
        ak = rng.uniform(-0.5, 1.5)
        wk = rng.uniform(0.05, 0.2)
        c = c + ak * np.exp(-((X - xk[0]) ** 2 + (Z - xk[1]) ** 2) / (2 * wk**2))
    return np.clip(c, 1.5, 4.5)


def medium_layered(g, seed=3, n_layers=20, amp_h=3.0):
    """c3: seeded horizontal layers with sinusoidally undulating interfaces."""
    X, Z = g.interior_xz()
    rng = np.random.default_rng(seed)
    vel = rng.uniform(1.5, 5.5, size=n_layers)
    below = np.zeros(X.shape, dtype=np.int64)
    for k in range(1, n_layers):
        kappa = rng.uniform(1.0, 4.0)
        phi = rng.uniform(0.0, 2 * np.pi)
        zk = k * g.Lz / n_layers + amp_h * g.h * np.sin(2 * np.pi * kappa * X / g.Lx + phi)
        below += (Z > zk).astype(np.int64)
    return vel[below]


def medium_faulted(g, seed=4, n_faults=6):
    """c4: linear gradient 1.5->4.5 with depth, signed dipping-fault jumps, clip,
    and a c=4.5 elliptic lens."""
    X, Z = g.interior_xz()
    rng = np.random.default_rng(seed)
    c = 1.5 + 3.0 * Z / g.Lz
    for _ in range(n_faults):
        xk = rng.uniform(0.1, 0.9) * g.Lx
        zk = rng.uniform(0.1, 0.9) * g.Lz
        th = np.deg2rad(rng.uniform(20.0, 70.0))
        side = rng.choice([-1.0, 1.0])
        sign = rng.choice([-1.0, 1.0])
        jump = rng.uniform(0.3, 1.0)
        c = c + sign * jump * (side * ((X - xk) * np.sin(th) - (Z - zk) * np.cos(th)) > 0)
    c = np.clip(c, 1.5, 4.5)
    lens = ((X - 0.5 * g.Lx) / 0.15) ** 2 + ((Z - 0.6 * g.Lz) / 0.05) ** 2 <= 1.0
    return np.where(lens, 4.5, c)


# ---- sources -----------------------------------------------------------------


def source_point(g, fx, fz, amp=1.0):
    f = np.zeros((g.nz_ext, g.nx_ext), dtype=np.complex128)
    px = min(max(int(round(fx * (g.nx + 1))), 1), g.nx)
    qz = min(max(int(round(fz * (g.nz + 1))), 1), g.nz)
    f[g.n_pml + qz - 1, g.n_pml + px - 1] = amp / g.h**2
    return f


def source_gaussian(g, fx, fz, sigma):
    f = np.zeros((g.nz_ext, g.nx_ext), dtype=np.complex128)
    z = g.z_coords()[g.n_pml:g.n_pml + g.nz]
    X, Z = np.meshgrid(g.x_coords(), z)
    x0, z0 = fx * g.Lx, fz * g.Lz
    f[g.n_pml:g.n_pml + g.nz, :] = (np.exp(-((X - x0) ** 2 + (Z - z0) ** 2) / (2 * sigma**2))
                                    / (2 * np.pi * sigma**2))
    return f


def source_random(g, seed):
    rng = np.random.default_rng(seed)
    f = np.zeros((g.nz_ext, g.nx_ext), dtype=np.complex128)
    shape = (g.nz, g.nx_ext)
    f[g.n_pml:g.n_pml + g.nz, :] = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return f


# ---- configurations ------------------------------------------------------------

CASES = ["c1", "c2", "c3", "c3r", "c4", "c4r", "c5"]
FIXTURES = ["fx_tiny", "fx_l2", "fx_uneven", "fx_plr", "fx_plr_odd", "fx_extrap", "fx_extrap_plr"]


def config(name: str) -> CaseConfig:
    if name == "c1":
        g = Geometry(200, 200, 20)
        return CaseConfig(name, g, medium_homogeneous(g), 4, 2 * np.pi * 20,
                          [("gauss", source_gaussian(g, 0.5, 0.1, 2 * g.h))], None, 1e-9,
                          "homogeneous c=1, 200^2+20 PML, omega=2pi*20, L=4, Gaussian source "
                          "sigma=2h, dense")
    if name in ("c2", "c5"):
        g = Geometry(400, 400, 30)
        c = medium_bumps(g)
        omega = 2 * np.pi * c.min() / (10 * g.h)
        if name == "c2":
            return CaseConfig(name, g, c, 8, omega, [("point", source_point(g, 0.5, 0.1))], None,
                              1e-9, "12 seeded Gaussian bumps (rng 2), 400^2+30 PML, 10 ppw, L=8, "
                              "point source, dense")
        src = [(f"point{s}", source_point(g, (s + 0.5) / 64, 0.05)) for s in range(64)]
        return CaseConfig(name, g, c, 8, omega, src, None, 1e-9,
                          "c2 medium and layering, 64 point sources at depth 0.05 (multi-RHS batch)")
    if name in ("c3", "c3r"):
        g = Geometry(800, 800, 40) if name == "c3" else Geometry(160, 160, 16)
        c = medium_layered(g)
        omega = 2 * np.pi * c.min() / (8 * g.h)
        L = 16 if name == "c3" else 4
        note = ("20 seeded layers (rng 3) with 3h undulation, 800^2+40 PML, 8 ppw, L=16, point "
                "source, PLR eps 1e-9 r_max 32" if name == "c3" else
                "reduced c3: layered medium 160^2+16 PML, 8 ppw, L=4, PLR eps 1e-9 r_max 32")
        return CaseConfig(name, g, c, L, omega, [("point", source_point(g, 0.5, 0.1))],
                          (1e-9, 32), 1e-9, note)
    if name in ("c4", "c4r"):
        g = Geometry(1600, 800, 40) if name == "c4" else Geometry(400, 200, 20)
        c = medium_faulted(g)
        omega = 2 * np.pi * c.min() / (8 * g.h)
        L = 32 if name == "c4" else 8
        return CaseConfig(name, g, c, L, omega, [("point", source_point(g, 0.5, 0.0))],
                          (1e-9, 32), 1e-9,
                          f"faulted gradient medium with lens (rng 4), {g.nx}x{g.nz}+{g.n_pml} PML, "
                          f"8 ppw, L={L}, surface point source, PLR eps 1e-9 r_max 32")
    # ---- small fixtures (tests/golden) ----
    if name == "fx_tiny":
        g = Geometry(8, 9, 3)
        return CaseConfig(name, g, medium_gradient(g), 3, 4.0, [("rand", source_random(g, 7))],
                          None, 1e-10, "reference test_solver.py tiny geometry: 8x9, L=3, "
                          "n_pml=3, omega=4, gradient")
    if name == "fx_l2":
        g = Geometry(12, 12, 4)
        return CaseConfig(name, g, medium_gradient(g), 2, 6.0,
                          [("point", source_point(g, 0.4, 0.3))], None, 1e-10,
                          "L=2 edge case (no kernel-bearing sweep steps)")
    if name == "fx_uneven":
        g = Geometry(10, 19, 4)
        return CaseConfig(name, g, medium_gradient(g), 4, 7.0,
                          [("point", source_point(g, 0.5, 0.7))], None, 1e-10,
                          "uneven layers 5,5,5,4 (remainder to the front), L=4")
    if name == "fx_plr":
        g = Geometry(40, 40, 10)
        return CaseConfig(name, g, medium_gradient(g), 4, 9.0,
                          [("point", source_point(g, 0.5, 0.25))], (1e-9, 4), 1e-10,
                          "PLR with real quadtree splits: m=60, r_max=4 (min leaf 8), L=4")
    if name == "fx_plr_odd":
        g = Geometry(37, 30, 8)
        return CaseConfig(name, g, medium_layered(g, seed=5, n_layers=5, amp_h=1.0), 3, 11.0,
                          [("point", source_point(g, 0.3, 0.5))], (1e-6, 3), 1e-10,
                          "PLR with odd m=53 (floor-first splits), eps 1e-6 (rank-deficient "
                          "leaves), L=3")
    if name == "fx_extrap":
        g = Geometry(30, 30, 10)
        return CaseConfig(name, g, medium_homogeneous(g), 3, 9.0,
                          [("point", source_point(g, 0.4, 0.6))], None, 1e-10,
                          "extrapolation variant (reference test_solver.py pipeline geometry: 30^2, "
                          "L=3, n_pml=10, omega=9, homogeneous), dense", variant="extrapolation")
    if name == "fx_extrap_plr":
        g = Geometry(40, 40, 10)
        return CaseConfig(name, g, medium_gradient(g), 4, 9.0,
                          [("point", source_point(g, 0.5, 0.25))], (1e-9, 4), 1e-10,
                          "extrapolation variant with PLR Green's blocks and dense E blocks "
                          "(mixed operator), m=60, r_max=4, L=4", variant="extrapolation")
    raise KeyError(f"unknown case {name!r}")
