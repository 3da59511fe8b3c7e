#!/usr/bin/env python
"""Benchmark of the B200 Polylla core (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A "step" is one pass of the whole hot path over one
mesh: polylla_build_halfedges -> polylla_label -> polylla_generate ->
polylla_get_polygons (CSR), inputs resident in HBM, no host sync inside the step.
Default workload: BASELINE config 3 (10M random points, Delaunay, ~20M triangles) --
the mesh the north_star's roofline target is stated on; its inputs (400 MB) and
working set (~1.7 GB) exceed the 126 MB L2, so no flush is needed between steps.

value      : input triangles/s, kernel-only, whole job (sum over ranks / max time)
e2e        : the same from pinned HOST buffers through polylla.HostPipeline (per mesh: H2D of
             xy+tri, the four C-ABI calls, D2H of CSR + origin/twin/next; the upload of mesh
             i+1 overlaps the download of mesh i), wall clock; `single_call_ms` = one
             synchronous polylla_run_host call, for reference
roofline   : dominant kernel group, algorithmic bytes / its live CUDA-event time
cpu_baseline: the CPU oracle (oracle/, 1 thread) on a bounded sample, rank 0 at N=1
--impl reference: the oracle as the reference arm (each step a bounded sample).
Under torchrun (N > 1) every rank converts its own mesh (weak scaling, no collective
on the data path); the max device time over ranks is all-reduced through NCCL.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2403_14723_b200 import batch  # noqa: E402

METRIC = "input triangles/sec (kernel-only pipeline build->label->generate->CSR, 1 mesh per GPU)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config: 1 tiny grid, 2 1M random, 3 10M random (default), 4 capacity, 5 batch")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the C-ABI calls eagerly instead of a CUDA graph")
    ap.add_argument("--order", default="morton", choices=["morton", "shuffled"],
                    help="triangle order of configs 2/3 (sensitivity rows): generator Morton order or shuffled")
    ap.add_argument("--no-pcie", action="store_true")
    ap.add_argument("--sort", action="store_true",
                    help="POLYLLA_BUILD_SORT: the build orders the triangles by Morton cell first (any input order)")
    ap.add_argument("--no-row-hint", action="store_true",
                    help="grid configs: contiguous 2,048-triangle build tiles instead of the row-stride grid tiling")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def workload(cfg: int, rank: int, world: int, device, order: str = "morton"):
    """Synthetic input of BASELINE config `cfg` for this rank (recipes: DESIGN.md 'Input
    recipe').  Returns (description, scaling, [mesh dicts with xy/tri device tensors and,
    for the e2e leg, a host generator])."""
    if cfg in (1, 2, 3):
        if cfg == 1:
            fn = lambda: synth.grid(32, 0.2, 1)  # noqa: E731
            name = "config1: jittered 32x32 grid (a=0.2), 1 mesh per GPU"
        else:
            n = 1_000_000 if cfg == 2 else 10_000_000
            fn = lambda: (lambda xy, tri: (xy, reorder(tri, order)))(*synth.random_delaunay(n, cfg + 1000 * rank))  # noqa: E731
            name = (f"config{cfg}: {n // 1_000_000}M random points, Delaunay ({order}-ordered triangles: "
                    f"{'centroid Morton order of the generator' if order == 'morton' else 'seeded random permutation'})"
                    f", 1 mesh per GPU")
        xy, tri = fn()
        m = dict(xy=torch.from_numpy(xy).to(device), tri=torch.from_numpy(tri).to(device), host=lambda: (xy, tri),
                 xy_np=xy, tri_np=tri, row_stride=2 * 31 if cfg == 1 else 0)
        return name, "weak", [m]
    if cfg == 4:
        xy, tri = synth.grid_device(16000, 0.2, 4 + 1000 * rank, device=device)
        name = "config4: jittered 16000x16000 grid (256M vertices, 512M triangles), generated on device, 1 per GPU"
        return name, "weak", [dict(xy=xy, tri=tri, host=None, row_stride=2 * 15999)]
    metas = [mm for mm in batch.config5_meshes() if mm["index"] in set(batch.shard(64, rank, world))]
    out = []
    for mm in metas:
        xy, tri = synth.grid_device(mm["s"], mm["a"], mm["seed"], device=device)
        out.append(dict(xy=xy, tri=tri, meta=mm, row_stride=2 * (mm["s"] - 1),
                        host=(lambda mm=mm: synth.grid(mm["s"], mm["a"], mm["seed"]))))
    name = ("config5: batch of 64 independent 2000x2000 grids (4M vertices each; 32 jittered a=0.2 + 32 regular "
            "Alg. 13), mesh i on rank i mod N, generated on device (excluded from timing)")
    return name, "strong", out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s from B200_PROFILING.md (MEASURED_PEAKS.json absent)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in names.items():
                    if r & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def alg_bytes(T, V, P, L, c=None):
    """Algorithmic bytes per launch of each kernel group (DESIGN.md section 6 states each
    model).  "pipeline" is SURVEY.md 8(d)'s B_alg = 60T + 16V + 12L + 4P, the method's
    compulsory HBM traffic for one mesh; the group models split the same accounting over
    the kernels (what each must read or write once).  c: the mesh's polylla counts."""
    c = c or {}
    n_left, n_def = c.get("n_leftover", 0), c.get("n_deferred", 0)
    n_sdef, tips, B = c.get("n_seed_deferred", 0), c.get("n_tips", 0), c.get("n_border", 0)
    tiles = (T + 2047) // 2048
    mean_loop = L / P if P else 0.0
    return {
        "pipeline": 60 * T + 16 * V + 12 * L + 4 * P,
        # B_alg's build rows: tri in (12T), origin/twin/next out (36T),
        # the FP64 coordinates once (16V)
        "k_tile": 48 * T + 16 * V,
        # per leftover: key + id in (12 B), twin out (4 B), border ranking re-reads id + twin (8 B)
        "k_left_match": 24 * n_left,
        # per border half-edge: blist, twin[e], origin[target] in; twin[e], twin[b], origin[b], vmap out
        "k_border_scan": 28 * B + 8 * tiles,
        # per border half-edge: origin[b], twin[b], origin[twin], vmap x2, origin[nx] in; next out
        "k_border_next": 28 * B,
        # per deferred half-edge: id, twin, Lcode x2 in, next out, + one rotation step (twin, Lcode x2)
        "k_label_fixup": 22 * n_def,
        # per tip: the degree walk about v (~6 twins) + middle-edge steps, F1/SDB words, and the
        # re-rewire of the two touched vertices (~2 x 6 x (twin + F1 + next))
        "k_repair": 96 * tips,
        # per global seed: F1 word + landing, then the loop walk (next per step), len/C/wlen out
        "k_seed_walk": int(n_sdef * (16 + 4 * mean_loop)),
        # C, wlen and F1 words in (12 B per 32 half-edges), per-tile sums
        "k_canon_scan": (12 * 3 * T) // 32 + 24 * tiles,
        # C bits + len at the canonical seeds in, next + origin along the loops, seeds +
        # offsets + loops out
        "k_extract": (3 * T) // 8 + 4 * P + 8 * L + 4 * P + 4 * (P + 1) + 4 * L,
    }


def src_hash():
    """Hash of the CUDA sources: ties a committed ncu traffic figure to this build."""
    import hashlib
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2403_14723_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh")):
            h.update(open(os.path.join(d, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "polylla.h"), "rb").read())
    return h.hexdigest()[:16]


def ncu_traffic(kernel: str, cfg: int):
    """dram__bytes_read + write per launch of `kernel`, from the committed `ncu --set full`
    capture of this build (profiles/ncu_traffic.json, written by
    profiles/tools/ncu_traffic.py with the source hash it was captured on); None if the
    capture is of other sources."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("src_hash") != src_hash():
            return None
        return d.get(f"config{cfg}", {}).get(kernel)
    except Exception:
        return None


def host_cpu():
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def _pinned_one_core(fn):
    """Run fn() with this thread pinned to one CPU (the taskset -c of SURVEY.md 8(d))."""
    try:
        old = os.sched_getaffinity(0)
        cpu = min(old)
        os.sched_setaffinity(0, {cpu})
    except (AttributeError, OSError):
        old, cpu = None, None
    try:
        return fn(), cpu
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)


def cpu_oracle_baseline(xy, tri):
    """Time the CPU oracle (built on this host with -O3 -march=native -ffp-contract=off,
    one thread pinned to one core) on a bounded sample of the workload (rank 0, N = 1)."""
    import oracle
    oracle.use_native()
    T = tri.shape[0]
    if T <= 25_000_000:
        sample_xy, sample_tri, what = xy, tri, f"the full bench mesh ({T} triangles), 1 run"
    else:
        n = 2_000_000
        sample_xy, sample_tri = xy, np.ascontiguousarray(tri[:n])
        what = f"the first {n} triangles of the bench mesh (a contiguous block of it), 1 run"
    t0 = time.perf_counter()
    o, cpu = _pinned_one_core(lambda: oracle.run(sample_xy, sample_tri))
    dt = time.perf_counter() - t0
    return {"value": sample_tri.shape[0] / dt, "unit": "triangles/s", "cores": 1, "kind": "oracle",
            "sample": what, "seconds": dt, "phases_s": o["times"], "pinned_cpu": cpu,
            "build": "gcc -O3 -march=native -ffp-contract=off (on this host)", "host": host_cpu()}


def reference_arm(args, ws, rank):
    """--impl reference: the CPU oracle, unmodified, as the reference arm: each step runs
    the oracle (one thread pinned to one core, -O3 -march=native) on a bounded sample of
    the SAME workload -- the first n triangles of the bench mesh (triangles come in Morton
    order, so this is a compact block of the mesh), n sized so the run ends in ~3 min."""
    if rank != 0:
        return
    import oracle
    oracle.use_native()
    steps, warm = args.steps, args.warmup
    name, xy, tri = host_workload(args.config, args.order)
    # calibrate on a small block of the same mesh
    nc = min(tri.shape[0], 200_000)
    t0 = time.perf_counter()
    _pinned_one_core(lambda: oracle.run(xy, np.ascontiguousarray(tri[:nc])))
    rate = nc / (time.perf_counter() - t0)
    budget = 150.0 / max(1, steps + warm)  # seconds per step
    n = int(min(tri.shape[0], max(2_000, 0.7 * rate * budget)))
    stri = np.ascontiguousarray(tri[:n])
    for _ in range(warm):
        _pinned_one_core(lambda: oracle.run(xy, stri))
    t0 = time.perf_counter()
    for _ in range(steps):
        _, cpu = _pinned_one_core(lambda: oracle.run(xy, stri))
    dt = time.perf_counter() - t0
    v = n * steps / dt
    what = (f"the first {n} of the {tri.shape[0]} triangles of the bench mesh ({name}) per step"
            if n < tri.shape[0] else f"the full bench mesh ({name}) per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "triangles/s", "n_gpus": ws,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64/i32", "data": "synthetic",
        "config": {"workload": name, "sample": what},
        "cpu_baseline": {"value": v, "unit": "triangles/s", "cores": 1, "kind": "oracle", "sample": what,
                         "pinned_cpu": cpu, "build": "gcc -O3 -march=native -ffp-contract=off",
                         "host": host_cpu()},
        "e2e": {"value": v, "unit": "triangles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def host_workload(cfg: int, order: str = "morton"):
    """The host copy of a single-mesh workload (configs 1-3; 4 and 5 use a 2000-grid)."""
    if cfg == 1:
        xy, tri = synth.grid(32, 0.2, 1)
        return "config1: jittered 32x32 grid (a=0.2)", xy, tri
    if cfg in (2, 3):
        n = 1_000_000 if cfg == 2 else 10_000_000
        xy, tri = synth.random_delaunay(n, cfg)
        tri = reorder(tri, order)
        return f"config{cfg}: {n // 1_000_000}M random points, Delaunay ({order} triangle order)", xy, tri
    xy, tri = synth.grid(2000, 0.2, 1000)
    return "config5 mesh 0: jittered 2000x2000 grid (a=0.2)", xy, tri


def reorder(tri, order: str):
    """Triangle order of the input (a sensitivity row of SURVEY.md 8(d)): "morton" is the
    generator's order (centroid Morton code); "shuffled" a seeded random permutation (the
    worst case for tile-local twin matching: almost every twin crosses tiles)."""
    if order == "morton":
        return tri
    perm = np.random.default_rng(12345).permutation(tri.shape[0])
    return np.ascontiguousarray(tri[perm])


def pcie_bandwidth(dev, nbytes=256 << 20, reps=5):
    """Pinned host <-> device copy bandwidth (GB/s), each direction alone (CUDA events)."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {}
    for name, (dst, src) in (("h2d_gbs", (d, h)), ("d2h_gbs", (h, d))):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(dev)
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[name] = nbytes / (best * 1e-3) / 1e9
    out["bytes_per_copy"] = nbytes
    return out


def main():
    args = parse()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, ws, rank)
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    from paper_2403_14723_b200 import polylla as pp

    dev = torch.device("cuda", local if ws > 1 else 0)
    if ws > 1:
        import torch.distributed as dist
    name, scaling, meshes = workload(args.config, rank, ws, dev, args.order)
    Vmax = max(m["xy"].shape[0] for m in meshes)
    Tmax = max(m["tri"].shape[0] for m in meshes)
    # grid inputs (row-major Alg. 13 triangle lists) pass their row stride 2(s-1): the build
    # then tiles 16-row x 128-triangle patches (polylla_build_halfedges_ex)
    R0 = 0 if args.no_row_hint or args.sort else meshes[0].get("row_stride", 0)
    SORT = bool(args.sort)
    if R0:
        name += f"; build tiles: 16 x 128-triangle patches (row stride hint {R0})"
    if SORT:
        name += "; build tiles over the Morton-cell order of the triangle centroids (POLYLLA_BUILD_SORT, in the timed step)"
    wsp = pp.alloc_workspace(Vmax, Tmax, dev, row_stride=R0, sort=SORT)
    offsets = torch.empty(Tmax + 1, dtype=torch.int32, device=dev)
    loops = torch.empty(3 * Tmax, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    launches = [0]

    def convert(m):
        ctx = pp.build_halfedges(m["xy"], m["tri"], wsp, stream, row_stride=R0, sort=SORT)
        pp.label(ctx, stream)
        pp.generate(ctx, stream)
        pp.get_polygons(ctx, offsets, loops, stream=stream)
        return ctx

    def step_eager():
        n = 0
        for m in meshes:
            ctx = convert(m)
            n += pp.launch_count(ctx)
            pp.destroy(ctx)
        launches[0] = n

    step = step_eager

    # A batch (config 5) converts its independent meshes on two streams with their own
    # workspaces and outputs, so one mesh's latency-bound tail kernels overlap the next
    # mesh's k_tile; the step ends when both streams have finished (joined on `stream`).
    lanes = None
    if len(meshes) > 1:
        n_lanes = int(os.environ.get("POLYLLA_BENCH_LANES", "2"))
        lanes = [dict(stream=stream, ws=wsp, offsets=offsets, loops=loops)] + [
            dict(stream=torch.cuda.Stream(device=dev), ws=pp.alloc_workspace(Vmax, Tmax, dev, row_stride=R0, sort=SORT),
                 offsets=torch.empty(Tmax + 1, dtype=torch.int32, device=dev),
                 loops=torch.empty(3 * Tmax, dtype=torch.int32, device=dev)) for _ in range(n_lanes - 1)]

        def step_batch():
            n = 0
            start = torch.cuda.Event()
            start.record(stream)
            for ln in lanes[1:]:
                ln["stream"].wait_event(start)
            for i, m in enumerate(meshes):
                ln = lanes[i % len(lanes)]
                s_ = ln["stream"]
                ctx = pp.build_halfedges(m["xy"], m["tri"], ln["ws"], s_, row_stride=R0, sort=SORT)
                pp.label(ctx, s_)
                pp.generate(ctx, s_)
                pp.get_polygons(ctx, ln["offsets"], ln["loops"], stream=s_)
                n += pp.launch_count(ctx)
                pp.destroy(ctx)
            for ln in lanes[1:]:
                done = torch.cuda.Event()
                done.record(ln["stream"])
                stream.wait_event(done)
            launches[0] = n

        step = step_batch

    # correctness gate + per-mesh counts (and a checksum of each CSR for cross-rank logs)
    stats = []
    for m in meshes:
        ctx = convert(m)
        c = pp.get_counts(ctx, stream)
        pp.destroy(ctx)
        P, L = c["n_polygons"], c["n_loop_entries"]
        m["counts"] = c
        ck = batch.loop_checksum(offsets[:P + 1], loops[:L])
        stats.append([m.get("meta", {}).get("index", rank), c["n_triangles"], P, L, c["n_tips"], c["n_border"], ck])
    local_T = sum(m["tri"].shape[0] for m in meshes)
    local_V = sum(m["xy"].shape[0] for m in meshes)
    local_P = sum(m["counts"]["n_polygons"] for m in meshes)
    local_L = sum(m["counts"]["n_loop_entries"] for m in meshes)

    graphs = None
    if not args.no_graph and len(meshes) == 1:
        # the whole step as one CUDA graph launch (same kernels, same stream order)
        graphs = [pp.GraphStep(m["xy"], m["tri"], wsp, offsets, loops, stream, row_stride=R0, sort=SORT)
                  for m in meshes]

        def step():
            for g in graphs:
                g.replay()
            launches[0] = sum(g.launches for g in graphs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local if ws > 1 else 0) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ms_total = batch.max_time(ev0.elapsed_time(ev1), dev, ws)
    tot = torch.tensor([float(local_T), float(local_P), float(local_V), float(local_L)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    all_T, all_P = float(tot[0].item()), float(tot[1].item())
    ms_step = ms_total / args.steps
    value = all_T * args.steps / (ms_total / 1e3)
    n_meshes_total = 64 if args.config == 5 else ws
    table = batch.gather_stats(torch.tensor(stats, dtype=torch.int64, device=dev), n_meshes_total, ws)
    for m in meshes:  # the counts must not change between runs (determinism)
        ctx = convert(m)
        c = pp.get_counts(ctx, stream)
        pp.destroy(ctx)
        assert c["status"] == 0 and c["n_polygons"] == m["counts"]["n_polygons"]

    # ---- live per-kernel times (CUDA events recorded by the library on `stream`; eager
    # launches, since events cannot be recorded from inside a replayed graph)
    pp.profile_enable(True)
    prof_steps = max(3, min(args.steps, 30 if args.config != 5 else 3))
    for _ in range(prof_steps):
        step_eager()
    prof = pp.profile_read()
    pp.profile_enable(False)
    per_launch = {k: ms / cnt for k, (ms, cnt) in prof.items()}
    prof_step_ms = sum(ms for ms, _ in prof.values()) / prof_steps
    nm = len(meshes)
    # algorithmic bytes per launch (one mesh per launch; meshes of a batch have equal size)
    ab = alg_bytes(local_T // nm, local_V // nm, local_P // nm, local_L // nm, meshes[0]["counts"])
    peak, peak_src = load_peaks()
    # the dominant kernel group: the largest share of the step (every group has a byte model)
    groups = {k: v for k, v in per_launch.items() if k in ab}
    missing = sorted(k for k in per_launch if k not in ab)
    top = max(groups, key=lambda k: groups[k] * prof[k][1])
    achieved = ab[top] / (per_launch[top] * 1e-3) / 1e9
    traffic = ncu_traffic(top, args.config)
    roof = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": ab[top],
            "kernel_ms": per_launch[top], "share_of_step": per_launch[top] * prof[top][1] / prof_steps / prof_step_ms,
            "peak_source": peak_src, "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes of this "
                                                        "source hash)" if traffic else "no capture of this build",
            "groups_without_model": missing}
    group_roof = {k: {"ms": per_launch[k] * prof[k][1] / prof_steps, "alg_bytes": ab[k],
                      "frac": ab[k] / (per_launch[k] * 1e-3) / 1e9 / peak} for k in groups}
    pipe_gbs = ab["pipeline"] * nm / (ms_step * 1e-3) / 1e9  # per GPU
    pipeline_roof = {"alg_bytes_per_step_per_gpu": ab["pipeline"] * nm, "achieved": pipe_gbs, "peak": peak,
                     "frac": pipe_gbs / peak, "frac_of_8TBs_nominal": pipe_gbs / 8000.0}

    # ---- end to end from pinned HOST buffers through the public API: HostPipeline
    # (H2D of xy/tri, build -> label -> generate -> CSR, D2H of CSR + origin/twin/next for
    # every mesh; upload of mesh i+1 overlaps the download of mesh i on full-duplex PCIe)
    e2e = None
    if not args.no_e2e and all(m.get("host") is not None for m in meshes):
        e_steps = max(2, min(args.e2e_steps, 10 if args.config != 5 else 1))
        hosts = []
        for m in meshes:
            xy_h, tri_h = m["host"]()
            hosts.append((torch.from_numpy(xy_h).pin_memory(), torch.from_numpy(tri_h).pin_memory()))
        inputs = [hosts[i % len(hosts)] for i in range(e_steps * len(hosts))]
        pipe = pp.HostPipeline(Vmax, Tmax, arrays=True, device=dev)
        outs = [pp.alloc_host_outputs(Tmax, arrays=True, pin=True) for _ in range(2)]
        out_list = [outs[i % 2] for i in range(len(inputs))]
        pipe.run(inputs[:2], out_list[:2])  # warm-up (first-touch of the pinned buffers)
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        cnts = pipe.run(inputs, out_list)
        torch.cuda.synchronize(dev)
        e_s = batch.max_time((time.perf_counter() - t0) * 1e3, dev, ws) / 1e3
        h2d = sum(16 * x.shape[0] + 12 * t.shape[0] for x, t in inputs) // e_steps
        d2h = sum(4 * (c["n_polygons"] + 1) + 4 * c["n_loop_entries"] + 12 * c["n_halfedges"] for c in cnts) // e_steps
        e2e = {"value": all_T * e_steps / e_s, "unit": "triangles/s", "ms_per_step": 1e3 * e_s / e_steps,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": "polylla.HostPipeline over the C ABI (pinned host in/out; CSR + origin/twin/next "
                      "returned; H2D of mesh i+1 overlapped with D2H of mesh i; wall clock, max over ranks)"}
        # the unpipelined single call, for reference
        r_ms = 0.0
        xy_h, tri_h = hosts[0]
        o1 = pp.alloc_host_outputs(Tmax, arrays=True, pin=True)
        pp.run_host(xy_h.numpy(), tri_h.numpy(), wsp, pinned=o1, stream=stream)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(3):
            pp.run_host(xy_h.numpy(), tri_h.numpy(), wsp, pinned=o1, stream=stream)
        torch.cuda.synchronize(dev)
        e2e["single_call_ms"] = 1e3 * (time.perf_counter() - t0) / 3
        assert cnts[-1]["n_polygons"] == meshes[(len(inputs) - 1) % len(meshes)]["counts"]["n_polygons"]

    if e2e is not None and not args.no_pcie:
        e2e["pcie"] = pcie_bandwidth(dev)
        e2e["pcie"]["copy_bound_ms_per_step"] = 1e3 * max(e2e["h2d_bytes_per_step"] / (e2e["pcie"]["h2d_gbs"] * 1e9),
                                                            e2e["d2h_bytes_per_step"] / (e2e["pcie"]["d2h_gbs"] * 1e9))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        if meshes[0].get("host") is not None:
            hx, ht = meshes[0]["host"]()
        else:
            hx, ht = synth.grid(2000, 0.2, 4)
        cpu = cpu_oracle_baseline(hx, ht)

    if rank == 0:
        c0 = meshes[0]["counts"]
        out = {
            "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64/i32", "data": "synthetic",
            "config": {"workload": name, "meshes": n_meshes_total, "T_total": int(all_T), "P_total": int(all_P),
                       "per_mesh_rank0": {"V": meshes[0]["xy"].shape[0], "T": meshes[0]["tri"].shape[0],
                                          "P": c0["n_polygons"], "L": c0["n_loop_entries"], "H": c0["n_halfedges"],
                                          "tips": c0["n_tips"], "leftover_halfedges": c0["n_leftover"],
                                          "deferred_halfedges": c0["n_deferred"],
                                          "deferred_seeds": c0["n_seed_deferred"]},
                       "l2": "no flush: per-step inputs and working set exceed the 126 MB L2" if args.config >= 3
                             else "small working set: L2-resident between steps (reported, not the headline)"},
            "polygons_per_s": all_P * args.steps / (ms_total / 1e3),
            "roofline": roof, "pipeline_roofline": pipeline_roof, "group_roofline": group_roof,
            "kernels_ms_per_step": {k: ms / prof_steps for k, (ms, _) in prof.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches[0] * args.steps,
            "launch_mode": ("cuda_graph (one graph launch per step)" if graphs else
                            f"eager, meshes alternating over {len(lanes)} streams" if lanes else "eager"),
            "clocks": clk.summary(),
            "mesh_table_head": table[:4].tolist(),
        }
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
