"""Input generators: recipe properties (CPU) and host/device bit-identity (GPU)."""
import math

import numpy as np
import pytest

import synth


def test_grid_shapes_and_orientation():
    xy, tri = synth.grid(5)
    assert xy.shape == (25, 2) and tri.shape == (32, 3)
    # Alg. 13 vertex k at (k div s, k mod s); every triangle is CW (reading R10)
    assert xy[7].tolist() == [1.0, 2.0]
    p = xy[tri]
    ar = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
    assert np.all(ar < 0)


def test_jitter_bounds_and_fixed_boundary():
    s, a = 40, 0.2
    xy, _ = synth.grid(s, a, 3)
    base, _ = synth.grid(s)
    d = xy - base
    assert np.abs(d).max() <= a
    ij = np.arange(s * s)
    border = (ij // s == 0) | (ij // s == s - 1) | (ij % s == 0) | (ij % s == s - 1)
    assert np.all(d[border] == 0) and np.all(np.abs(d[~border]) > 0)


def test_random_delaunay_recipe():
    n = 20000
    xy, tri = synth.random_delaunay(n, 4)
    assert xy.shape == (n, 2)
    assert xy[:4].tolist() == [[0, 0], [1, 0], [1, 1], [0, 1]]
    assert len(np.unique(xy, axis=0)) == n  # duplicates were redrawn
    # lattice coordinates, and nothing left inside the snapping band (R18)
    assert np.all(xy * 2 ** 24 == np.round(xy * 2 ** 24))
    delta = 1 / math.sqrt(n)
    inner = (xy > 0) & (xy < 1)
    assert np.all((xy[inner] >= delta - 2 ** -24) & (xy[inner] <= 1 - delta + 2 ** -24))
    # CCW triangles covering the unit square, Euler for a disk
    p = xy[tri]
    ar = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
    assert np.all(ar > 0) and abs(ar.sum() / 2 - 1.0) < 1e-12
    # determinism
    xy2, tri2 = synth.random_delaunay(n, 4)
    assert np.array_equal(xy, xy2) and np.array_equal(tri, tri2)


def test_random_delaunay_empty_circumcircle_small():
    """Delaunay property by brute force on a small instance."""
    xy, tri = synth.random_delaunay(300, 9)
    P = (xy * 2 ** 24).astype(np.int64)
    for a, b, c in tri.tolist():
        A, B, C = P[a], P[b], P[c]
        d = P - C  # translate; exact integer in-circle determinant via Python ints
        ad, bd = A - C, B - C
        for q in range(len(P)):
            if q in (a, b, c):
                continue
            qx, qy = int(P[q][0] - C[0]), int(P[q][1] - C[1])
            ax, ay, bx, by = int(ad[0]) - qx, int(ad[1]) - qy, int(bd[0]) - qx, int(bd[1]) - qy
            cx, cy = -qx, -qy
            det = (ax * ax + ay * ay) * (bx * cy - cx * by) + (bx * bx + by * by) * (cx * ay - ax * cy) + \
                  (cx * cx + cy * cy) * (ax * by - bx * ay)
            assert det <= 0
        del d


@pytest.mark.gpu
def test_device_grid_matches_host():
    import torch
    for s, a, seed in [(2, 0.0, 0), (37, 0.2, 5), (200, 0.2, 1000)]:
        xd, td = synth.grid_device(s, a, seed)
        xh, th = synth.grid(s, a, seed)
        torch.cuda.synchronize()
        assert np.array_equal(xd.cpu().numpy(), xh)
        assert np.array_equal(td.cpu().numpy(), th)
