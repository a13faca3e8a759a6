"""GPU offline stage against the host offline stage.

The device extraction of a layer's interface Green's blocks (multi-column
sparse triangular solves, reference local_solver.py:112-135) and the batched
quadtree compression (reference plr.py:200-236) must reproduce the host
restatement -- itself pinned bitwise to the reference on the fixtures
(tests/test_offline.py) -- to the rounding of a different factorization order
and SVD driver.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _layer(nx=56, n_layer=11, n_pml=7, ppw=9.0):
    from paper_1410_5910_b200.offline.layers import Layer, layer_operator
    from paper_1410_5910_b200.offline.local import factor_layer
    h = 1.0 / (nx + 1)
    omega = 2 * np.pi / (ppw * h)
    rng = np.random.default_rng(5)
    c = 1.0 + 0.5 * rng.random((n_layer + 2 * n_pml, nx + 2 * n_pml))
    m_tilde = 1.0 / c**2
    host = Layer(nx, n_layer, h, n_pml, omega, m_tilde)
    op = layer_operator(nx, n_layer, h, n_pml, omega, m_tilde)
    fac = factor_layer(op, n_layer + 2 * n_pml, nx + 2 * n_pml)
    return host, fac, (nx, n_layer, n_pml, h)


def test_greens_blocks_match_host():
    import torch
    from paper_1410_5910_b200.offline.gpu import DeviceLayer
    host, fac, (nx, n_layer, n_pml, h) = _layer()
    depths = (0, 1, n_layer, n_layer + 1)
    pairs = [(j, k) for j in depths for k in depths]
    ref = host.greens(pairs)
    dev = DeviceLayer(fac, n_layer + 2 * n_pml, nx + 2 * n_pml, n_layer, n_pml, h, "cuda")
    for chunk in (None, 16):  # all columns at once, and in column chunks
        got = dev.greens(pairs, chunk=chunk)
        torch.cuda.synchronize()
        for p in pairs:
            g = got[p].cpu().numpy()
            assert g.shape == ref[p].shape
            err = np.linalg.norm(g - ref[p]) / np.linalg.norm(ref[p])
            assert err < 1e-10, (p, chunk, err)


def test_batched_quadtree_matches_host():
    import torch
    from paper_1410_5910_b200.offline.compress import plr_leaves
    from paper_1410_5910_b200.offline.gpu import plr_leaves_gpu
    rng = np.random.default_rng(7)
    n = 150  # odd splits on the way down (150 -> 75 -> 37 / 38)
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    blocks = []
    for s in range(3):  # Green's-function-like kernels: smooth off the diagonal
        d = np.abs(i - j) + 0.5 + s
        blocks.append(np.exp(1j * (0.9 + 0.2 * s) * d) / np.sqrt(d)
                      + 1e-3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
                      * (np.abs(i - j) < 4))
    r_max, eps = 8, 1e-7
    got = plr_leaves_gpu([torch.from_numpy(b).cuda() for b in blocks], r_max, eps)
    for b, leaves in zip(blocks, got):
        ref = plr_leaves(b, r_max, eps)
        assert [(r0, c0, u.shape, v.shape) for r0, c0, u, v in leaves] == \
               [(r0, c0, u.shape, v.shape) for r0, c0, u, v in ref]
        rebuilt = np.zeros_like(b)
        for r0, c0, u, v in leaves:
            rebuilt[r0:r0 + u.shape[0], c0:c0 + v.shape[1]] = u @ v
        ref_rebuilt = np.zeros_like(b)
        for r0, c0, u, v in ref:
            ref_rebuilt[r0:r0 + u.shape[0], c0:c0 + v.shape[1]] = u @ v
        assert np.linalg.norm(rebuilt - ref_rebuilt) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("compress_on,workers", [("host", 2), ("host", 1), ("cuda", 1)])
def test_gpu_built_operator_equals_host_built(compress_on, workers):
    """A whole reduced-c3 case through build_operator(device="cuda"): same
    entry table, same leaf structure, kernels and right-hand sides to rounding
    (compression on the host workers as the blocks arrive, or batched on the GPU)."""
    from paper_1410_5910_b200.offline.build import build_operator
    m_h, a_h = build_operator("c3r", workers=1, sources=True)
    m_g, a_g = build_operator("c3r", workers=workers, sources=True, device="cuda",
                              compress_on=compress_on)
    assert m_h["kernel_format"] == m_g["kernel_format"] == "plr"
    np.testing.assert_array_equal(a_h["entries"], a_g["entries"])
    # leaf table rows: (kernel, row_off, col_off, rows, cols, rank, u_off, vt_off)
    lh, lg = a_h["leaves"], a_g["leaves"]
    np.testing.assert_array_equal(lh, lg)
    # per-leaf products agree (the factors themselves are unique up to phases)
    fh, fg = a_h["factors"], a_g["factors"]
    worst = 0.0
    for row in lh[:: max(1, len(lh) // 200)]:
        mm, kk, r, uo, vo = (int(v) for v in row[3:8])
        ph = fh[uo:uo + mm * r].reshape(mm, r) @ fh[vo:vo + r * kk].reshape(r, kk)
        pg = fg[uo:uo + mm * r].reshape(mm, r) @ fg[vo:vo + r * kk].reshape(r, kk)
        worst = max(worst, np.linalg.norm(ph - pg) / max(np.linalg.norm(ph), 1e-300))
    assert worst < 1e-6, worst
    err = np.linalg.norm(a_h["rhs"] - a_g["rhs"]) / np.linalg.norm(a_h["rhs"])
    assert err < 1e-9, err
