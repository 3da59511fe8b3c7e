"""Grid tiling (polylla_build_halfedges_ex with a row stride R): k_tile takes 16-row x
128-triangle patches of a row-major triangle list instead of 2,048 consecutive triangles.
A performance hint only -- the conversion must be the same bits for ANY R that divides T,
so every output (origin/twin/next/prev, the stage bit-vectors, seeds, CSR, per-triangle
polygon and region ids) is compared element by element with the CPU oracle:

  - Alg. 13 grids (R = 2(s-1)), jittered and regular, with s chosen
    so that the last tile column and the last tile band are partial (R and T/R not
    multiples of 128 and 16) and meshes smaller than one band;
  - a random Delaunay mesh (Morton-ordered) and a shuffled one with R = a divisor of T
    that has nothing to do with the geometry: only the grouping of triangles changes."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import bits_to_bool

pytestmark = pytest.mark.gpu


def _check(xy, tri, R, sort=False):
    from paper_2403_14723_b200 import polylla as pp
    T = tri.shape[0]
    assert sort or T % R == 0
    ref = oracle.run(xy, tri)
    res = pp.run(torch.from_numpy(xy).cuda(), torch.from_numpy(np.ascontiguousarray(tri)).cuda(), row_stride=R,
                 debug=True, prev=True, regions=True, sort=sort)
    assert (res["H"], res["P"], res["L"], res["n_tips"]) == (ref["H"], ref["P"], ref["L"], ref["n_tips"])
    for k in ("origin", "twin", "next", "prev", "seeds", "offsets", "loops"):
        np.testing.assert_array_equal(res[k].cpu().numpy(), ref[k], err_msg=k)
    np.testing.assert_array_equal(res["lcode"].cpu().numpy(), ref["lcode"])
    for k in ("frontier0", "frontier1"):
        np.testing.assert_array_equal(bits_to_bool(res[k], 3 * T), ref[k][:3 * T].astype(bool), err_msg=k)
    np.testing.assert_array_equal(np.nonzero(bits_to_bool(res["seed_bits"], 3 * T))[0], ref["seeds0"])
    np.testing.assert_array_equal(res["next_pre"].cpu().numpy(), ref["next_pre"])
    np.testing.assert_array_equal(res["poly_of_tri"].cpu().numpy(), oracle.triangle_polygons(ref))
    np.testing.assert_array_equal(res["region_of_tri"].cpu().numpy(), oracle.triangle_regions(ref))
    return res


@pytest.mark.parametrize("s,a", [(6, 0.2), (30, 0.2), (67, 0.0), (67, 0.2), (131, 0.2), (200, 0.0), (301, 0.2)])
def test_grid_tiles_alg13(s, a):
    xy, tri = synth.grid(s, a, 7)
    res = _check(xy, tri, 2 * (s - 1))
    if s >= 67:  # the point of the hint: few leftovers (a 16 x 128 patch cuts ~3% of its half-edges)
        assert res["n_leftover"] < 0.06 * 3 * tri.shape[0]


@pytest.mark.parametrize("which", ["smallest", "whole"])
def test_grid_tiles_degenerate_strides(which):
    """Strides that make every tile partial: the smallest divisor > 1 of T (rows of a few
    triangles: 16 x R patches) and R = T (one row: 1 x 128 patches)."""
    xy, tri = synth.random_delaunay(4000, 19)
    T = tri.shape[0]
    R = T if which == "whole" else next(d for d in range(2, T + 1) if T % d == 0)
    _check(xy, tri, R)


@pytest.mark.parametrize("shuffle", [False, True])
def test_grid_tiles_any_stride(shuffle):
    xy, tri = synth.random_delaunay(30000, 12)
    T = tri.shape[0]
    if shuffle:
        tri = np.ascontiguousarray(tri[np.random.default_rng(4).permutation(T)])
    R = next(d for d in range(300, T + 1) if T % d == 0)  # a divisor of T unrelated to the mesh
    _check(xy, tri, R)


@pytest.mark.parametrize("name", ["shuffled", "random", "grid", "fan", "tie", "holes"])
def test_sorted_tiles(name):
    """The sorted tiling (POLYLLA_BUILD_SORT: tiles over the Morton-cell order of the
    triangle centroids, for any input order), bit-exact vs the oracle."""
    from test_gpu_parity import _grid_with_holes
    if name == "shuffled":
        xy, tri = synth.random_delaunay(40000, 13)
        tri = np.ascontiguousarray(tri[np.random.default_rng(5).permutation(tri.shape[0])])
    elif name == "random":
        xy, tri = synth.random_delaunay(30000, 14)
    elif name == "grid":
        xy, tri = synth.grid(120, 0.2, 2)
    elif name == "holes":
        xy, tri = _grid_with_holes()
    else:
        xy, tri = {"fan": synth.fixture_fan, "tie": synth.fixture_tie_lattice}[name]()
    res = _check(xy, tri, 0, sort=True)
    if name == "shuffled":  # the point of it: few leftovers although the input order is random
        assert res["n_leftover"] < 0.10 * 3 * tri.shape[0]
