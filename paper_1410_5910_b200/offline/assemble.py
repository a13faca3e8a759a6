"""The polarized "jump" system as an entry table (host offline), restated.

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
"""

from __future__ import annotations

import numpy as np

__all__ = ["polarized_table", "polarized_rhs", "sweep_order"]

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


def sweep_order(L):
    """Down rows (T_{2i-1}, B_{2i-1}), then up rows (B_{2i}, T_{2i}) (trace_system.py:353-365)."""
    nt = 2 * L - 2
    down = [v for i in range(1, L) for v in (2 * i - 2, nt + 2 * i - 2)]
    up = [v for i in range(1, L) for v in (nt + 2 * i - 1, 2 * i - 1)]
    return np.array(down + up, dtype=np.int64)


def polarized_table(n_c, h):
    """Entry table of the jump system for layer offsets n_c (length L+1).

    Returns (entries (E,3) int64 [row, col, kernel|-1], coefs (E,2) complex
    [scale, eye], keys [(layer, target depth, source depth)] per kernel id,
    perm).
    """
    L = len(n_c) - 1
    if L < 2:
        raise ValueError("interface system needs at least two layers")
    thick = [int(n_c[ell] - n_c[ell - 1]) for ell in range(1, L + 1)]
    nt = 2 * L - 2
    col = {"dn": lambda i, s: 2 * (i - 1) + s, "up": lambda i, s: nt + 2 * (i - 1) + s}
    acc = {}

    def add(row, c, key, sign, eye):
        cur = acc.setdefault((row, c), [None, 1.0 + 0j, 0j])
        if key is not None:
            if cur[0] is not None:
                raise ValueError(f"block ({row},{c}) assigned two kernels")
            cur[0], cur[1] = key, complex(sign / h)
        cur[2] += complex(eye)

    for i in range(1, L):
        for row, items, owner, target in (
                (2 * (i - 1), _T_TOP, i, "n"), (nt + 2 * (i - 1), _B_TOP, i, "n1"),
                (2 * i - 1, _T_BOT, i + 1, "1"), (nt + 2 * i - 1, _B_BOT, i + 1, "0")):
            n_own = thick[owner - 1]
            depth = {"1": 1, "0": 0, "n": n_own, "n1": n_own + 1}
            for half, d, slot, src, sign, eye in items:
                ii = i + d
                if ii < 1 or ii > L - 1:
                    continue
                # sources on the far interface use the owning layer's own depths
                key = None if src is None else (owner, depth[target], depth[src])
                add(row, col[half](ii, slot), key, sign, eye)
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


def polarized_rhs(newtons, n_c):
    """[-(N^i at n, N^{i+1} at 1)...; -(N^i at n+1, N^{i+1} at 0)...] (trace_system.py:311-326, 475-484)."""
    L = len(n_c) - 1
    top, bot = [], []
    for i in range(1, L):
        n = n_c[i] - n_c[i - 1]
        top += [newtons[i - 1][n], newtons[i][1]]
        bot += [newtons[i - 1][n + 1], newtons[i][0]]
    return np.concatenate([-np.concatenate(top), -np.concatenate(bot)])
