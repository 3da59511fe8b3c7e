"""BASELINE config 4 (the capacity probe: jittered 16000 x 16000 grid, V = 256M,
T = 511,936,002, H = 1,535,872,002 < 2^31) bit-exact against the CPU oracle.

The oracle needs ~100 GB of host memory (its [H] arrays trimmed to the known H =
3T + 4(s-1) through oracle.run(hcap=...)) and ~3.5 minutes on one core (measured on the
B200 host: 202 s, profiles/r02/config4_oracle_bitexact.txt), so the test is skipped on a
host with less than 150 GB of available memory.  The device-side invariant check of
the same mesh runs too (tests/test_gpu_parity.py::test_config4_capacity_invariants)."""
import gc
import os
import time

import numpy as np
import pytest
import torch

import oracle
import synth

def _mem_available_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return 0.0


pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _host_info():
    mem = [l for l in open("/proc/meminfo") if l.startswith(("MemTotal", "MemAvailable"))]
    cpu = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")
    return f"host: {cpu}, {os.cpu_count()} logical CPUs; " + "; ".join(l.strip() for l in mem)


def _eq_chunked(dev_arr, host_arr, name, chunk=1 << 27):
    n = host_arr.shape[0]
    assert dev_arr.numel() >= n, name
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        h = torch.from_numpy(np.ascontiguousarray(host_arr[a:b])).cuda()
        if not torch.equal(dev_arr[a:b], h):
            bad = int(torch.nonzero(dev_arr[a:b] != h)[0, 0]) + a
            raise AssertionError(f"{name}[{bad}]: gpu {int(dev_arr[bad])} oracle {int(host_arr[bad])}")
        del h


@pytest.mark.skipif(_mem_available_gb() < 150, reason="needs ~100 GB of host RAM (150 GB available)")
def test_config4_bit_exact_vs_oracle():
    """Both build tilings of the GPU path -- contiguous 2,048-triangle tiles and the grid
    tiling that bench.py uses for this row-major input (row stride 2(s-1)) -- against one
    oracle run, every array element by element."""
    from paper_2403_14723_b200 import polylla as pp
    print(_host_info(), flush=True)
    s = 16000
    t0 = time.time()
    xy, tri = synth.grid(s, 0.2, 4)
    T = tri.shape[0]
    assert T == 511_936_002
    H = 3 * T + 4 * (s - 1)
    print(f"generated in {time.time() - t0:.0f} s", flush=True)
    t0 = time.time()
    ref = oracle.run(xy, tri, hcap=H)
    print(f"oracle: {time.time() - t0:.0f} s, phases {ref['times']}", flush=True)
    for R in (0, 2 * (s - 1)):
        xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
        ws = pp.alloc_workspace(xy.shape[0], T, row_stride=R)
        t0 = time.time()
        ctx = pp.build_halfedges(xd, td, ws, row_stride=R)
        pp.label(ctx)
        pp.generate(ctx)
        c = pp.get_counts(ctx)
        assert c["n_halfedges"] == H
        P, L = c["n_polygons"], c["n_loop_entries"]
        offsets = torch.empty(P + 1, dtype=torch.int32, device="cuda")
        loops = torch.empty(L, dtype=torch.int32, device="cuda")
        pp.get_polygons(ctx, offsets, loops)
        assert pp.get_counts(ctx)["status"] == 0
        torch.cuda.synchronize()
        print(f"gpu (row stride {R}): {time.time() - t0:.1f} s (incl. first launches) P={P} L={L} "
              f"tips={c['n_tips']} leftovers={c['n_leftover']}", flush=True)
        del xd, td
        assert (ref["H"], ref["P"], ref["L"], ref["n_tips"]) == (H, P, L, c["n_tips"])
        v = pp.get_views(ctx)
        view = lambda k, n: pp.view_tensor(ctx, v[k], n, torch.int32)  # noqa: E731
        for k in ("origin", "twin", "next"):
            _eq_chunked(view(k, H), ref[k], k)
        _eq_chunked(view("seeds", P), ref["seeds"], "seeds")
        _eq_chunked(offsets, ref["offsets"], "offsets")
        _eq_chunked(loops, ref["loops"], "loops")
        lc = pp.view_tensor(ctx, v["lcode"], T, torch.uint8)
        _eq_chunked(lc, ref["lcode"], "lcode")
        print(f"config 4 bit-exact (row stride {R}): origin/twin/next [{H}], lcode [{T}], seeds [{P}], offsets, "
              f"loops [{L}]", flush=True)
        pp.destroy(ctx)
        del ws, offsets, loops, v, lc, view, ctx  # (the Context holds the workspace tensor)
        gc.collect()
        torch.cuda.empty_cache()


def test_int32_ceiling_invariants():
    """The int32 ceiling (PAPER.md L55's capacity question): a
    jittered grid with s = 18,919 has T = 715,781,448 and H = 3T + 4(s-1) = 2,147,420,016
    <= 2^31 - 1 half-edges -- the largest grid signed 32-bit ids would address, and the
    largest the default worst-case layout (6T <= 2^32 - 2) accepts.  Workspace ~144 GB +
    14 GB of input on the 178 GB device; checked by the properties that hold at any size,
    on the device.  (Past it: tests/test_gpu_capacity.py, unsigned ids, bounded layout.)"""
    from paper_2403_14723_b200 import polylla as pp
    from test_gpu_parity import device_invariants
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # (other tests' cached blocks: this one needs ~158 GB of the 178)
    s = 18919
    T = 2 * (s - 1) ** 2
    H = 3 * T + 4 * (s - 1)
    assert H <= 2**31 - 1 < 3 * 2 * s * s + 4 * s  # (s + 1 would overflow)
    xy, tri = synth.grid_device(s, 0.2, 5)
    ws = pp.alloc_workspace(xy.shape[0], T)
    ctx = pp.build_halfedges(xy, tri, ws)
    pp.label(ctx)
    pp.generate(ctx)
    c = pp.get_counts(ctx)
    assert c["n_halfedges"] == H and c["n_border"] == 4 * (s - 1)
    P, L = c["n_polygons"], c["n_loop_entries"]
    offsets = torch.empty(P + 1, dtype=torch.int32, device="cuda")
    loops = torch.empty(L, dtype=torch.int32, device="cuda")
    pp.get_polygons(ctx, offsets, loops)
    assert pp.get_counts(ctx)["status"] == 0
    v = pp.get_views(ctx)
    view = lambda k, n: pp.view_tensor(ctx, v[k], n, torch.int32)  # noqa: E731
    got = device_invariants(xy, tri, view("origin", H), view("twin", H), view("next", H), offsets, loops,
                            view("seeds", P))
    assert got == P
    print(f"int32 ceiling s={s}: T={T} H={H} P={P} L={L} tips={c['n_tips']}", flush=True)
    pp.destroy(ctx)
