"""The paper's kernel sequence (polylla_label_generate_paper: LLK, LFK, LSK, LEK, CaK, SFK,
OSK, Scan -- SURVEY.md §8(f) NEXT-2, the ablation) against the CPU oracle, element by
element: it must give exactly what the default path gives."""
import numpy as np
import pytest

import oracle
import synth
from test_gpu_parity import _grid_with_holes, _wheels, bits_to_bool, gpu_run

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(4)
    xy, tri = synth.random_delaunay(20000, 41)
    return {
        "square": synth.fixture_square(), "triangle": synth.fixture_triangle(), "fan": synth.fixture_fan(),
        "tie": synth.fixture_tie_lattice(), "grid": synth.grid(64), "jittered": synth.grid(150, 0.2, 3),
        "random": synth.random_delaunay(50000, 6), "shuffled": (xy, np.ascontiguousarray(tri[rng.permutation(tri.shape[0])])),
        "holes": _grid_with_holes(), "wheels": _wheels(),
    }


@pytest.mark.parametrize("name", list(_cases()))
def test_paper_sequence_bit_exact(name):
    xy, tri = _cases()[name]
    ref = oracle.run(xy, tri)
    res = gpu_run(xy, tri, paper=True, prev=True, debug=True, regions=True)
    T = tri.shape[0]
    assert res["H"] == ref["H"] and res["n_tips"] == ref["n_tips"]
    for k in ("origin", "twin", "next", "prev"):
        np.testing.assert_array_equal(res[k].cpu().numpy(), ref[k], err_msg=k)
    for k in ("seeds", "offsets", "loops"):
        np.testing.assert_array_equal(res[k].cpu().numpy(), ref[k], err_msg=k)
    np.testing.assert_array_equal(bits_to_bool(res["frontier0"], 3 * T), ref["frontier0"][:3 * T].astype(bool))
    np.testing.assert_array_equal(bits_to_bool(res["frontier1"], 3 * T), ref["frontier1"][:3 * T].astype(bool))
    np.testing.assert_array_equal(res["poly_of_tri"].cpu().numpy(), oracle.triangle_polygons(ref))
    np.testing.assert_array_equal(res["region_of_tri"].cpu().numpy(), oracle.triangle_regions(ref))


@pytest.mark.slow
def test_paper_sequence_config2():
    xy, tri = synth.random_delaunay(1_000_000, 2)
    ref = oracle.run(xy, tri)
    res = gpu_run(xy, tri, paper=True)
    for k in ("next", "seeds", "offsets", "loops"):
        np.testing.assert_array_equal(res[k].cpu().numpy(), ref[k], err_msg=k)


@pytest.mark.parametrize("s,a", [(64, 0.0), (150, 0.2)])
def test_paper_sequence_after_grid_tiling(s, a):
    """The ablation after a grid-tiled build (row-stride hint): the paper's kernels read
    only the global arrays, so the result is the oracle's."""
    xy, tri = synth.grid(s, a, 3)
    ref = oracle.run(xy, tri)
    res = gpu_run(xy, tri, paper=True, prev=True, regions=True, row_stride=2 * (s - 1))
    for k in ("origin", "twin", "next", "prev", "seeds", "offsets", "loops"):
        np.testing.assert_array_equal(res[k].cpu().numpy(), ref[k], err_msg=k)
    np.testing.assert_array_equal(res["poly_of_tri"].cpu().numpy(), oracle.triangle_polygons(ref))
