"""The polarized system as an entry table (host offline), restated.

For every interface i = 1..L-1 the reference fills four block rows of the
doubled system (trace_system.py:400-459):

  T_{2i-1}  layer i at depth n          B_{2i-1}  layer i at depth n+1
  T_{2i}    layer i+1 at depth 1        B_{2i}    layer i+1 at depth 0

with +-(1/h) G_l[target, source] blocks and exact -I identities.  Here the
rows are written as data: each item is (column half, interface offset,
slot, source depth selector, sign, eye).  Entries accumulate exactly like
BlockInterfaceMatrix.add (trace_system.py:196-207): one kernel per block, eye
terms summed.  Kernel ids are assigned by first appearance over the entries
sorted by (row, col), which is how the reference's operator is captured.

Two variants, as ``assemble_polarized`` (trace_system.py:368-472): "jump"
completes the B rows with outside-depth relations; "extrapolation" with the
one-sided trace steppers E (trace_system.py:329-350, 460-464): row B_{2i-1}
is E_down(layer i) x_dn(i,0) - x_dn(i,1), row B_{2i} is -x_up(i,0) +
E_up(layer i+1) x_up(i,1), each E at scale 1.0 and never compressed.
"""

from __future__ import annotations

import numpy as np

__all__ = ["polarized_table", "polarized_rhs", "sweep_order", "extrapolator", "extrapolator_pairs"]

# (half, d_interface, slot, source, sign, eye); source in {"1","0","n","n1"}
# meaning local depth 1, 0, n_src, n_src+1 of the layer that owns the row;
# rows coupling to interface i-1 / i+1 exist only when that interface does.
_T_TOP = [("dn", -1, 0, "1", +1, 0), ("dn", -1, 1, "0", -1, 0),
          ("up", -1, 0, "1", +1, 0), ("up", -1, 1, "0", -1, 0),
          ("dn", 0, 0, None, 0, -1),
          ("up", 0, 0, "n1", -1, -1), ("up", 0, 1, "n", +1, 0)]
_B_TOP = [("dn", -1, 0, "1", +1, 0), ("dn", -1, 1, "0", -1, 0),
          ("up", -1, 0, "1", +1, 0), ("up", -1, 1, "0", -1, 0),
          ("dn", 0, 1, None, 0, -1),
          ("up", 0, 0, "n1", -1, 0), ("up", 0, 1, "n", +1, 0)]
_T_BOT = [("dn", 0, 0, "1", +1, 0), ("dn", 0, 1, "0", -1, -1),
          ("up", 0, 1, None, 0, -1),
          ("dn", +1, 0, "n1", -1, 0), ("dn", +1, 1, "n", +1, 0),
          ("up", +1, 0, "n1", -1, 0), ("up", +1, 1, "n", +1, 0)]
_B_BOT = [("dn", 0, 0, "1", +1, 0), ("dn", 0, 1, "0", -1, 0),
          ("up", 0, 0, None, 0, -1),
          ("dn", +1, 0, "n1", -1, 0), ("dn", +1, 1, "n", +1, 0),
          ("up", +1, 0, "n1", -1, 0), ("up", +1, 1, "n", +1, 0)]
# extrapolation variant: E kernels (source "Edown"/"Eup"), scale 1.0
_B_TOP_EX = [("dn", 0, 0, "Edown", 1, 0), ("dn", 0, 1, None, 0, -1)]
_B_BOT_EX = [("up", 0, 0, None, 0, -1), ("up", 0, 1, "Eup", 1, 0)]
VARIANTS = ("jump", "extrapolation")


def extrapolator(num, den):
    """E with E @ den = num: a partially pivoted dense solve, never an explicit
    inverse (trace_system.py:329-350).  down: num = G(n+1, n), den = G(n, n);
    up: num = G(0, 1), den = G(1, 1) of the layer's own blocks."""
    return np.linalg.solve(den.T, num.T).T


def extrapolator_pairs(n, direction):
    """(target, source) Green's blocks an extrapolator needs: (num, den)."""
    return ((n + 1, n), (n, n)) if direction == "down" else ((0, 1), (1, 1))


def sweep_order(L):
    """Down rows (T_{2i-1}, B_{2i-1}), then up rows (B_{2i}, T_{2i}) (trace_system.py:353-365)."""
    nt = 2 * L - 2
    down = [v for i in range(1, L) for v in (2 * i - 2, nt + 2 * i - 2)]
    up = [v for i in range(1, L) for v in (nt + 2 * i - 1, 2 * i - 1)]
    return np.array(down + up, dtype=np.int64)


def polarized_table(n_c, h, variant="jump"):
    """Entry table of the polarized system for layer offsets n_c (length L+1).

    Returns (entries (E,3) int64 [row, col, kernel|-1], coefs (E,2) complex
    [scale, eye], keys per kernel id -- (layer, target depth, source depth)
    for a Green's block, (layer, "E", "down"|"up") for an extrapolator --
    perm).
    """
    if variant not in VARIANTS:
        raise ValueError(f"unknown polarized variant {variant!r}")
    L = len(n_c) - 1
    if L < 2:
        raise ValueError("interface system needs at least two layers")
    thick = [int(n_c[ell] - n_c[ell - 1]) for ell in range(1, L + 1)]
    nt = 2 * L - 2
    col = {"dn": lambda i, s: 2 * (i - 1) + s, "up": lambda i, s: nt + 2 * (i - 1) + s}
    acc = {}

    def add(row, c, key, scale, eye):
        cur = acc.setdefault((row, c), [None, 1.0 + 0j, 0j])
        if key is not None:
            if cur[0] is not None:
                raise ValueError(f"block ({row},{c}) assigned two kernels")
            cur[0], cur[1] = key, complex(scale)
        cur[2] += complex(eye)

    b_top, b_bot = (_B_TOP, _B_BOT) if variant == "jump" else (_B_TOP_EX, _B_BOT_EX)
    for i in range(1, L):
        for row, items, owner, target in (
                (2 * (i - 1), _T_TOP, i, "n"), (nt + 2 * (i - 1), b_top, i, "n1"),
                (2 * i - 1, _T_BOT, i + 1, "1"), (nt + 2 * i - 1, b_bot, i + 1, "0")):
            n_own = thick[owner - 1]
            depth = {"1": 1, "0": 0, "n": n_own, "n1": n_own + 1}
            for half, d, slot, src, sign, eye in items:
                ii = i + d
                if ii < 1 or ii > L - 1:
                    continue
                # sources on the far interface use the owning layer's own depths
                if src is None:
                    key, scale = None, 0.0
                elif src in ("Edown", "Eup"):
                    key, scale = (owner, "E", src[1:]), 1.0
                else:
                    key, scale = (owner, depth[target], depth[src]), sign / h
                add(row, col[half](ii, slot), key, scale, eye)
    items = sorted(acc.items())
    entries = np.zeros((len(items), 3), dtype=np.int64)
    coefs = np.zeros((len(items), 2), dtype=np.complex128)
    kid, keys = {}, []
    for n, ((r, c), (key, scale, eye)) in enumerate(items):
        k = -1
        if key is not None:
            if key not in kid:
                kid[key] = len(keys)
                keys.append(key)
            k = kid[key]
        entries[n] = (r, c, k)
        coefs[n] = (scale, eye)
    return entries, coefs, keys, sweep_order(L)


def polarized_rhs(newtons, n_c, variant="jump"):
    """[-(N^i at n, N^{i+1} at 1)...; -(N^i at n+1, N^{i+1} at 0)...] (trace_system.py:311-326,
    475-484); the extrapolation variant's bottom half is zero."""
    L = len(n_c) - 1
    top, bot = [], []
    for i in range(1, L):
        n = n_c[i] - n_c[i - 1]
        top += [newtons[i - 1][n], newtons[i][1]]
        bot += [newtons[i - 1][n + 1], newtons[i][0]]
    top = -np.concatenate(top)
    if variant == "extrapolation":
        return np.concatenate([top, np.zeros_like(top)])
    return np.concatenate([top, -np.concatenate(bot)])
