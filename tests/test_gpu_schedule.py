"""Schedule independence and fallback paths, element by element
against the CPU oracle:

  - compile-time variants (tests/variants.py): reversed tile order, other block sizes,
    a 384-thread k_tile without pointer jumping, and a build whose k_emit always takes
    the dense-tile branch and whose in-tile loop walks bail out after 3 steps (the
    global seed walk then closes almost every polygon);
  - run time: a workspace filled with random bytes, unrelated kernels (an L2-sized
    fill and a GEMM) launched on the same stream between the C-ABI calls.

Every output array (origin/twin/next/prev, stage bit-vectors, seeds, CSR) must be
bit-exact with the oracle in every variant."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import _grid_with_holes, _wheels, assert_parity
from variants import VARIANTS, build_variants

pytestmark = pytest.mark.gpu


def _meshes():
    rng = np.random.default_rng(3)
    xy, tri = synth.random_delaunay(20000, 17)
    shuf = np.ascontiguousarray(tri[rng.permutation(tri.shape[0])])
    return {
        "fan": synth.fixture_fan(),
        "tie": synth.fixture_tie_lattice(),
        "grid": synth.grid(100),
        "jittered": synth.grid(150, 0.2, 3),
        "random": synth.random_delaunay(30000, 5),
        "shuffled": (xy, shuf),
        "holes": _grid_with_holes(),
        "wheels": _wheels(),
    }


@pytest.fixture(scope="module")
def variant_paths():
    return build_variants()


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_variant_bit_exact(variant, variant_paths):
    from paper_2403_14723_b200 import polylla as pp
    prev = pp.set_library(variant_paths[variant])
    try:
        for name, (xy, tri) in _meshes().items():
            res, _ = assert_parity(xy, tri, invariants=False)
            if variant == "fallback" and name in ("random", "jittered"):
                assert res["n_seed_deferred"] > 0.5 * res["P"], name  # the global walk did the work
        # grid tiling (row-stride hint) under the same variant: partial tiles, arbitrary stride
        from test_gpu_grid_tiles import _check
        for s_, a_ in ((150, 0.2), (131, 0.0)):
            gx, gt = synth.grid(s_, a_, 3)
            _check(gx, gt, 2 * (s_ - 1))
        rx, rt = synth.random_delaunay(8000, 41)
        _check(rx, rt, next(d for d in range(100, rt.shape[0] + 1) if rt.shape[0] % d == 0))
    finally:
        pp.set_library(prev)


def test_garbage_workspace_and_interleaved_kernels():
    """Uninitialised workspace bytes and unrelated work between the calls must not change
    a single output (no kernel reads a workspace region it did not write this run)."""
    from paper_2403_14723_b200 import polylla as pp
    xy, tri = synth.random_delaunay(40000, 23)
    ref = oracle.run(xy, tri)
    T = tri.shape[0]
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    s = torch.cuda.Stream()
    junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    a = torch.randn(2048, 2048, device="cuda")
    for trial in range(2):
        ws = pp.alloc_workspace(xy.shape[0], T)
        g = torch.Generator(device="cuda").manual_seed(trial)
        ws.copy_(torch.randint(0, 256, ws.shape, dtype=torch.uint8, device="cuda", generator=g))
        torch.cuda.synchronize()

        def noise():
            with torch.cuda.stream(s):
                junk.fill_(trial + 1)
                torch.mm(a, a)

        with torch.cuda.stream(s):
            ctx = pp.build_halfedges(xd, td, ws, s)
            noise()
            pp.label(ctx, s)
            noise()
            pp.generate(ctx, s)
            noise()
            c = pp.get_counts(ctx, s)
            P, L, H = c["n_polygons"], c["n_loop_entries"], c["n_halfedges"]
            offs = torch.full((T + 1,), -7, dtype=torch.int32, device="cuda")
            loops = torch.full((3 * T,), -7, dtype=torch.int32, device="cuda")
            arr = {k: torch.full((H,), -7, dtype=torch.int32, device="cuda") for k in ("origin", "twin", "next", "prev")}
            pp.get_polygons(ctx, offs, loops, stream=s, **arr)
            pp.get_counts(ctx, s)
            pp.destroy(ctx)
        s.synchronize()
        assert H == ref["H"] and P == ref["P"] and L == ref["L"]
        np.testing.assert_array_equal(offs[:P + 1].cpu().numpy(), ref["offsets"])
        np.testing.assert_array_equal(loops[:L].cpu().numpy(), ref["loops"])
        for k in ("origin", "twin", "next", "prev"):
            np.testing.assert_array_equal(arr[k].cpu().numpy(), ref[k], err_msg=k)


def test_garbage_workspace_grid_tiling():
    """The grid tiling ORs its words into bit-vectors it zeroes first: a workspace of random
    bytes must not leak into any output."""
    from paper_2403_14723_b200 import polylla as pp
    s_ = 140
    xy, tri = synth.grid(s_, 0.2, 13)
    R = 2 * (s_ - 1)
    ref = oracle.run(xy, tri)
    T = tri.shape[0]
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    for trial in range(2):
        ws = pp.alloc_workspace(xy.shape[0], T, row_stride=R)
        g = torch.Generator(device="cuda").manual_seed(7 + trial)
        ws.copy_(torch.randint(0, 256, ws.shape, dtype=torch.uint8, device="cuda", generator=g))
        ctx = pp.build_halfedges(xd, td, ws, row_stride=R)
        pp.label(ctx)
        pp.generate(ctx)
        c = pp.get_counts(ctx)
        P, L, H = c["n_polygons"], c["n_loop_entries"], c["n_halfedges"]
        offs = torch.empty(P + 1, dtype=torch.int32, device="cuda")
        loops = torch.empty(L, dtype=torch.int32, device="cuda")
        arr = {k: torch.empty(H, dtype=torch.int32, device="cuda") for k in ("origin", "twin", "next", "prev")}
        pp.get_polygons(ctx, offs, loops, **arr)
        assert pp.get_counts(ctx)["status"] == 0
        np.testing.assert_array_equal(offs.cpu().numpy(), ref["offsets"])
        np.testing.assert_array_equal(loops.cpu().numpy(), ref["loops"])
        for k in ("origin", "twin", "next", "prev"):
            np.testing.assert_array_equal(arr[k].cpu().numpy(), ref[k], err_msg=k)
        pp.destroy(ctx)


def test_host_prev_pointer():
    """prev into a host buffer (pageable and pinned) goes through device
    scratch and a copy, and equals the oracle's prev."""
    from paper_2403_14723_b200 import polylla as pp
    xy, tri = synth.random_delaunay(20000, 29)
    ref = oracle.run(xy, tri)
    T = tri.shape[0]
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    for pinned in (False, True):
        ws = pp.alloc_workspace(xy.shape[0], T)
        ctx = pp.build_halfedges(xd, td, ws)
        pp.label(ctx)
        pp.generate(ctx)
        c = pp.get_counts(ctx)
        H = c["n_halfedges"]
        prev = torch.full((H,), -7, dtype=torch.int32, pin_memory=pinned)
        offs = torch.empty(T + 1, dtype=torch.int32, device="cuda")
        loops = torch.empty(3 * T, dtype=torch.int32, device="cuda")
        pp.get_polygons(ctx, offs, loops, prev=prev)
        assert pp.get_counts(ctx)["status"] == 0
        np.testing.assert_array_equal(prev.numpy(), ref["prev"])
        pp.destroy(ctx)
