"""Capacity beyond int32 (the capacity question of PAPER.md L55 and
the compact data structure of L1071).

Half-edge ids (twin, next, prev, seeds) and CSR offsets are unsigned 32-bit in the C ABI
(include/polylla.h): a mesh may have up to H = 2^32 - 2 half-edges, twice the int32
ceiling (s = 18,919 grid, tests/test_gpu_config4.py).  polylla_workspace_bytes_ex /
polylla_build_halfedges_ex size origin/twin/next by 3T + a border bound instead of 6T and
drop run_host's staging, which brings an s = 20,000 grid (T = 799,920,002,
H = 2,399,840,002 > 2^31 - 1) to ~101 GB of workspace.

  - small meshes: the bounded layout gives the oracle's arrays bit for bit, and a bound
    below B is reported (POLYLLA_E_WORKSPACE), never overrun;
  - the default layout of a mesh past the int32 range is refused synchronously
    (POLYLLA_E_INDEX_OVERFLOW: 6T > 2^32 - 2);
  - s = 20,000 regular Alg. 13 grid: EVERY entry of origin, twin,
    next, lcode, seeds, offsets and loops against the grid's closed form -- each polygon
    is its unit cell (Tables 2-3 "Rep = 0.0"; pinned against the oracle at small
    s by tests/test_oracle_pins.py) -- computed independently here, chunk by chunk;
  - s = 20,000 jittered grid (a = 0.2): the properties that hold at any size
    (test_gpu_parity.device_invariants, ids read unsigned)."""
import gc

import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import _pp, device_invariants, u32

pytestmark = pytest.mark.gpu

S_BIG = 20_000


def _free_gb():
    gc.collect()
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0] / 1e9


def _run(pp, xy, tri, max_border, staging=False, row_stride=0):
    T = tri.shape[0]
    ws = pp.alloc_workspace(xy.shape[0], T, max_border=max_border, staging=staging, row_stride=row_stride)
    ctx = pp.build_halfedges(xy, tri, ws, max_border=max_border, staging=staging, row_stride=row_stride)
    pp.label(ctx)
    pp.generate(ctx)
    return ws, ctx


@pytest.mark.parametrize("name", ["grid40", "random", "fan"])
def test_border_bound_layout_matches_oracle(name):
    """The bounded layout (3T + max_border entries, no staging) is the same conversion."""
    pp = _pp()
    xy, tri = {"grid40": lambda: synth.grid(40, 0.2, 3), "random": lambda: synth.random_delaunay(5000, 8),
               "fan": synth.fixture_fan}[name]()
    ref = oracle.run(xy, tri)
    B = ref["H"] - 3 * tri.shape[0]
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    ws, ctx = _run(pp, xd, td, max_border=B)
    assert ws.numel() < pp.workspace_bytes(xy.shape[0], tri.shape[0])
    c = pp.get_counts(ctx)
    H, P, L = c["n_halfedges"], c["n_polygons"], c["n_loop_entries"]
    assert (H, P, L) == (ref["H"], ref["P"], ref["L"])
    out = {k: torch.empty(n, dtype=torch.int32, device="cuda")
           for k, n in (("offsets", P + 1), ("loops", L), ("origin", H), ("twin", H), ("next", H), ("prev", H))}
    pp.get_polygons(ctx, out["offsets"], out["loops"], origin=out["origin"], twin=out["twin"], next=out["next"],
                    prev=out["prev"])
    assert pp.get_counts(ctx)["status"] == 0
    for k in ("offsets", "loops", "origin", "twin", "next", "prev"):
        np.testing.assert_array_equal(out[k].cpu().numpy(), ref[k], err_msg=k)
    pp.destroy(ctx)


def test_border_bound_too_small_is_reported():
    pp = _pp()
    xy, tri = synth.grid(30, 0.2, 2)  # B = 4 * 29
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    ws, ctx = _run(pp, xd, td, max_border=4 * 29 - 1)
    c = pp.get_counts(ctx, check=False)
    assert pp.STATUS[c["status"]] == "WORKSPACE"
    pp.destroy(ctx)
    ws, ctx = _run(pp, xd, td, max_border=4 * 29)
    assert pp.get_counts(ctx)["n_border"] == 4 * 29
    pp.destroy(ctx)


def test_default_layout_refuses_past_int32():
    """6T > 2^32 - 2: the worst-case layout of an s = 20,000 grid cannot be addressed; the
    call fails before touching the device (a 1-byte workspace is never read)."""
    pp = _pp()
    T = 2 * (S_BIG - 1) ** 2
    xy = torch.zeros((4, 2), dtype=torch.float64, device="cuda")
    tri = torch.zeros((1, 3), dtype=torch.int32, device="cuda")
    import ctypes
    h = ctypes.c_void_p()
    ws = torch.empty(256, dtype=torch.uint8, device="cuda")
    L = pp.lib()
    rc = L.polylla_build_halfedges(pp._ptr(xy), S_BIG * S_BIG, pp._ptr(tri), T, pp._ptr(ws), ws.numel(), None,
                                   ctypes.byref(h))
    assert pp.STATUS[rc] == "INDEX_OVERFLOW"
    rc = L.polylla_build_halfedges_ex(pp._ptr(xy), S_BIG * S_BIG, pp._ptr(tri), T, 4 * (S_BIG - 1), 0, 0,
                                      pp._ptr(ws), ws.numel(), None, ctypes.byref(h))
    assert pp.STATUS[rc] == "WORKSPACE"  # addressable; only the workspace is too small


def _closed_form_check(ctx, pp, s, offsets, loops, chunk=1 << 24):
    """Every array of the regular s x s Alg. 13 grid against its closed form.  Cell
    c = (i, j), i, j < s-1, lower-left vertex k = i s + j (vertex k at (k div s, k mod s));
    its triangles 2c, 2c+1 are (k, k+1, k+s+1) and (k, k+s+1, k+s), both CW, re-oriented
    (R10) to (k, k+s+1, k+1) and (k, k+s, k+s+1).  The diagonals 6c and 6c+5 are the
    longest edges (|d|^2 = 2 > 1); the legs are frontier; each cell is one polygon with
    canonical seed 6c+1 and loop (k+s+1, k+1, k, k+s) (next: 6c+1 -> 6c+2 -> 6c+3 ->
    6c+4 -> 6c+1; the diagonals keep next_in)."""
    n = s - 1
    P, T = n * n, 2 * n * n
    T3, H = 3 * T, 3 * T + 4 * n
    v = pp.get_views(ctx)
    view = lambda k, m, dt=torch.int32: pp.view_tensor(ctx, v[k], m, dt)  # noqa: E731
    origin, twin, nxt, seeds = view("origin", H), view("twin", H), view("next", H), view("seeds", P)
    lcode = view("lcode", T, torch.uint8)
    dev = origin.device
    for c0 in range(0, P, chunk):
        c1 = min(P, c0 + chunk)
        c = torch.arange(c0, c1, device=dev, dtype=torch.int64)
        i, j = c // n, c % n
        k = i * s + j
        e0 = 6 * c
        sl = slice(6 * c0, 6 * c1)
        exp_org = torch.stack([k, k + s + 1, k + 1, k, k + s, k + s + 1], 1).reshape(-1)
        assert torch.equal(origin[sl].long(), exp_org), "origin"
        exp_nxt = torch.stack([e0 + 1, e0 + 2, e0 + 3, e0 + 4, e0 + 1, e0 + 3], 1).reshape(-1)
        assert torch.equal(u32(nxt[sl]), exp_nxt), "next"
        tw = u32(twin[sl]).view(-1, 6)
        cell = lambda ii, jj: ii * n + jj  # noqa: E731
        assert torch.equal(tw[:, 0], e0 + 5) and torch.equal(tw[:, 5], e0), "twin (diagonals)"
        for col, ok, partner in ((1, j + 1 < n, 6 * cell(i, j + 1) + 3), (2, i >= 1, 6 * cell(i - 1, j) + 4),
                                 (3, j >= 1, 6 * cell(i, j - 1) + 1), (4, i + 1 < n, 6 * cell(i + 1, j) + 2)):
            assert torch.equal(tw[ok, col], partner[ok]), f"twin (leg {col})"
            assert bool(torch.all(tw[~ok, col] >= T3)), f"twin (border leg {col})"
        lc = lcode[2 * c0:2 * c1].long().view(-1, 2)
        assert bool(torch.all(lc[:, 0] == 0)) and bool(torch.all(lc[:, 1] == 2)), "lcode"
        assert torch.equal(u32(seeds[c0:c1]), e0 + 1), "seeds"
        assert torch.equal(u32(offsets[c0:c1]), 4 * c), "offsets"
        exp_loop = torch.stack([k + s + 1, k + 1, k, k + s], 1).reshape(-1)
        assert torch.equal(loops[4 * c0:4 * c1].long(), exp_loop), "loops"
    assert int(u32(offsets[P:P + 1])) == 4 * P
    # border half-edges [3T, H): twins interior and involutive, origin = target of the twin,
    # next a permutation of the border ids that continues at the twin's origin
    b = torch.arange(T3, H, device=dev)
    tb = u32(twin[T3:H])
    assert bool(torch.all(tb < T3)) and torch.equal(u32(twin[tb]), b)
    nb = u32(nxt[T3:H])
    assert torch.equal(torch.sort(nb).values, b)
    assert torch.equal(origin[nb], origin[tb])


@pytest.mark.slow
@pytest.mark.parametrize("tiling", ["contiguous", "grid"])
def test_regular_grid_beyond_int32_closed_form(tiling):
    pp = _pp()
    if _free_gb() < 140:
        pytest.skip("needs ~130 GB of free device memory")
    s = S_BIG
    n = s - 1
    T, P = 2 * n * n, n * n
    H = 3 * T + 4 * n
    assert H > 2**31 - 1 and H <= 2**32 - 2
    xy, tri = synth.grid_device(s, 0.0, 0)
    ws, ctx = _run(pp, xy, tri, max_border=4 * n, row_stride=2 * n if tiling == "grid" else 0)
    c = pp.get_counts(ctx)
    assert (c["n_halfedges"], c["n_border"], c["n_polygons"], c["n_loop_entries"], c["n_tips"]) == (
        H, 4 * n, P, 4 * P, 0)
    offsets = torch.empty(P + 1, dtype=torch.int32, device="cuda")
    loops = torch.empty(4 * P, dtype=torch.int32, device="cuda")
    pp.get_polygons(ctx, offsets, loops)
    assert pp.get_counts(ctx)["status"] == 0
    _closed_form_check(ctx, pp, s, offsets, loops)
    print(f"regular s={s} ({tiling} tiles): T={T} H={H} (> 2^31 - 1) P={P}: every array = the closed form",
          flush=True)
    pp.destroy(ctx)


@pytest.mark.slow
def test_jittered_grid_beyond_int32_invariants():
    pp = _pp()
    if _free_gb() < 140:
        pytest.skip("needs ~135 GB of free device memory")
    s = S_BIG
    n = s - 1
    T = 2 * n * n
    H = 3 * T + 4 * n
    xy, tri = synth.grid_device(s, 0.2, 20)
    ws, ctx = _run(pp, xy, tri, max_border=4 * n)
    c = pp.get_counts(ctx)
    assert c["n_halfedges"] == H > 2**31 - 1 and c["n_border"] == 4 * n
    P, L = c["n_polygons"], c["n_loop_entries"]
    offsets = torch.empty(P + 1, dtype=torch.int32, device="cuda")
    loops = torch.empty(L, dtype=torch.int32, device="cuda")
    pp.get_polygons(ctx, offsets, loops)
    assert pp.get_counts(ctx)["status"] == 0
    v = pp.get_views(ctx)
    view = lambda k, m: pp.view_tensor(ctx, v[k], m, torch.int32)  # noqa: E731
    got = device_invariants(xy, tri, view("origin", H), view("twin", H), view("next", H), offsets, loops,
                            view("seeds", P))
    assert got == P
    print(f"jittered s={s}: T={T} H={H} P={P} L={L} tips={c['n_tips']}", flush=True)
    pp.destroy(ctx)
