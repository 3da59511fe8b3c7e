"""Thin Python binding of ``libpolylla.so`` (include/polylla.h), same names as the C ABI.

Argument marshalling only: every step of the conversion runs in the CUDA kernels of
the library.  PyTorch supplies device memory (the workspace and output tensors) and
streams.  There is no CPU fallback: importing works anywhere, but every call loads the
shared library and fails loudly if it is missing or no GPU is present.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POLYLLA_LIB") or os.path.join(_HERE, "libpolylla.so")  # override: A/B experiments

STATUS = {
    0: "OK", -1: "INVALID_ARGUMENT", -2: "DANGLING_INDEX", -3: "DEGENERATE_TRI",
    -4: "NON_MANIFOLD_EDGE", -5: "NON_MANIFOLD_VERTEX", -6: "INDEX_OVERFLOW", -7: "WORKSPACE",
    -8: "WALK_BOUND", -9: "UNSEEDED_LOOP", -10: "CALL_ORDER", -11: "CUDA", -12: "CAPACITY",
}

# every symbol include/polylla.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "polylla_workspace_bytes", "polylla_build_halfedges", "polylla_label", "polylla_generate",
    "polylla_get_counts", "polylla_get_polygons", "polylla_get_views", "polylla_set_debug",
    "polylla_run_host", "polylla_destroy", "polylla_status_string", "polylla_launch_count",
    "polylla_profile_enable", "polylla_profile_read", "polylla_get_triangle_polygons",
    "polylla_check_manifold", "polylla_get_triangle_regions", "polylla_label_generate_paper",
    "polylla_workspace_bytes_ex", "polylla_build_halfedges_ex",
)

WS_STAGING = 1  # POLYLLA_WS_STAGING
BUILD_SORT = 2  # POLYLLA_BUILD_SORT


class PolyllaError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        super().__init__(f"{where}: polylla status {code} ({STATUS.get(code, '?')})")
        self.code = code


class Counts(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "n_vertices", "n_triangles", "n_halfedges", "n_border", "n_polygons", "n_loop_entries",
        "n_tips", "n_flips", "n_leftover", "n_deferred", "n_seed_deferred")] + [("status", ctypes.c_int32),
                                                                               ("reserved", ctypes.c_int32)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_ if k != "reserved"}


class Views(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "origin", "twin", "next", "lcode", "frontier0", "frontier1", "seed_bits", "seeds", "tips")]


_LIB = None
_LIBS = {}


def set_library(path: str | None):
    """Use another build of the library (a flag variant, tests/variants.py) for the calls
    that follow; None restores the default.  Returns the previous path."""
    global _LIB, LIB_PATH
    prev = LIB_PATH
    LIB_PATH = path or os.path.join(_HERE, "libpolylla.so")
    _LIB = _LIBS.get(LIB_PATH)
    return prev


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32p = ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p
        L.polylla_workspace_bytes.restype = ctypes.c_size_t
        L.polylla_workspace_bytes.argtypes = [i64, i64]
        L.polylla_build_halfedges.restype = ctypes.c_int
        L.polylla_build_halfedges.argtypes = [vp, i64, vp, i64, vp, ctypes.c_size_t, vp, ctypes.POINTER(vp)]
        if hasattr(L, "polylla_build_halfedges_ex"):  # (older builds, loaded for A/B timing, lack it)
            L.polylla_workspace_bytes_ex.restype = ctypes.c_size_t
            L.polylla_workspace_bytes_ex.argtypes = [i64, i64, i64, ctypes.c_uint32, i64]
            L.polylla_build_halfedges_ex.restype = ctypes.c_int
            L.polylla_build_halfedges_ex.argtypes = [vp, i64, vp, i64, i64, ctypes.c_uint32, i64, vp,
                                                     ctypes.c_size_t, vp, ctypes.POINTER(vp)]
        for n in ("polylla_label", "polylla_generate", "polylla_check_manifold", "polylla_label_generate_paper"):
            getattr(L, n).restype = ctypes.c_int
            getattr(L, n).argtypes = [vp, vp]
        L.polylla_get_counts.restype = ctypes.c_int
        L.polylla_get_counts.argtypes = [vp, vp, ctypes.POINTER(Counts)]
        L.polylla_get_polygons.restype = ctypes.c_int
        L.polylla_get_polygons.argtypes = [vp, i32p, i64, i32p, i64, i32p, i32p, i32p, i32p, vp]
        L.polylla_get_triangle_polygons.restype = ctypes.c_int
        L.polylla_get_triangle_polygons.argtypes = [vp, i32p, vp]
        L.polylla_get_triangle_regions.restype = ctypes.c_int
        L.polylla_get_triangle_regions.argtypes = [vp, i32p, vp]
        L.polylla_get_views.restype = ctypes.c_int
        L.polylla_get_views.argtypes = [vp, ctypes.POINTER(Views)]
        L.polylla_set_debug.restype = ctypes.c_int
        L.polylla_set_debug.argtypes = [vp, vp]
        L.polylla_run_host.restype = ctypes.c_int
        L.polylla_run_host.argtypes = [vp, i64, vp, i64, vp, ctypes.c_size_t, vp, i64, vp, i64, vp, vp, vp, i64,
                                       ctypes.POINTER(Counts), vp]
        L.polylla_destroy.restype = None
        L.polylla_destroy.argtypes = [vp]
        L.polylla_status_string.restype = ctypes.c_char_p
        L.polylla_status_string.argtypes = [ctypes.c_int]
        L.polylla_launch_count.restype = ctypes.c_int64
        L.polylla_launch_count.argtypes = [vp]
        L.polylla_profile_enable.restype = None
        L.polylla_profile_enable.argtypes = [ctypes.c_int]
        L.polylla_profile_read.restype = ctypes.c_int
        L.polylla_profile_read.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        _LIB = _LIBS[LIB_PATH] = L
    return _LIB


def _stream(stream):
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check(rc, where):
    if rc != 0:
        raise PolyllaError(rc, where)


@dataclass
class Context:
    """A polylla_ctx plus the torch tensors it views (kept alive here)."""
    handle: ctypes.c_void_p
    xy: torch.Tensor
    tri: torch.Tensor
    workspace: torch.Tensor

    def __del__(self):
        if destroy is not None:  # (module globals are already cleared at interpreter exit)
            destroy(self)


def _flags(staging: bool, sort: bool) -> int:
    return (WS_STAGING if staging else 0) | (BUILD_SORT if sort else 0)


def workspace_bytes(n_vertices: int, n_triangles: int, max_border: int | None = None, staging: bool = True,
                    row_stride: int = 0, sort: bool = False) -> int:
    """polylla_workspace_bytes, or polylla_workspace_bytes_ex when a border bound, a row
    stride, sort=True or staging=False is given (the capacity path; grid or
    sorted tiling)."""
    if max_border is None and staging and not row_stride and not sort:
        return int(lib().polylla_workspace_bytes(n_vertices, n_triangles))
    mb = 3 * n_triangles if max_border is None else max_border
    return int(lib().polylla_workspace_bytes_ex(n_vertices, n_triangles, mb, _flags(staging, sort), row_stride))


def alloc_workspace(n_vertices: int, n_triangles: int, device="cuda", max_border: int | None = None,
                    staging: bool = True, row_stride: int = 0, sort: bool = False) -> torch.Tensor:
    return torch.empty(workspace_bytes(n_vertices, n_triangles, max_border, staging, row_stride, sort),
                       dtype=torch.uint8, device=device)


def build_halfedges(xy: torch.Tensor, tri: torch.Tensor, workspace: torch.Tensor, stream=None,
                    max_border: int | None = None, staging: bool = True, row_stride: int = 0,
                    sort: bool = False) -> Context:
    """polylla_build_halfedges; with a border bound, a row stride (row-major input: grid
    tiles), sort=True (any input order: tiles over the Morton-sorted triangles) or
    staging=False polylla_build_halfedges_ex over a workspace from
    alloc_workspace(..., max_border, staging, row_stride, sort) (the same arguments)."""
    if not (xy.is_cuda and tri.is_cuda and workspace.is_cuda):
        raise ValueError("xy, tri and workspace must be CUDA tensors")
    if xy.dtype != torch.float64 or tri.dtype != torch.int32 or not xy.is_contiguous() or not tri.is_contiguous():
        raise ValueError("xy must be contiguous float64 [V,2], tri contiguous int32 [T,3]")
    h = ctypes.c_void_p()
    if max_border is None and staging and not row_stride and not sort:
        rc = lib().polylla_build_halfedges(_ptr(xy), xy.shape[0], _ptr(tri), tri.shape[0], _ptr(workspace),
                                           workspace.numel(), _stream(stream), ctypes.byref(h))
    else:
        mb = 3 * tri.shape[0] if max_border is None else max_border
        rc = lib().polylla_build_halfedges_ex(_ptr(xy), xy.shape[0], _ptr(tri), tri.shape[0], mb,
                                              _flags(staging, sort), row_stride, _ptr(workspace),
                                              workspace.numel(), _stream(stream), ctypes.byref(h))
    _check(rc, "polylla_build_halfedges")
    return Context(h, xy, tri, workspace)


def check_manifold(ctx: Context, stream=None) -> None:
    """Opt-in exact non-manifold-edge check (polylla_check_manifold); the verdict arrives
    with the next get_counts."""
    _check(lib().polylla_check_manifold(ctx.handle, _stream(stream)), "polylla_check_manifold")


def label_generate_paper(ctx: Context, stream=None) -> None:
    """The paper's kernel sequence (LLK..OSK + Scan) instead of label + generate (ablation)."""
    _check(lib().polylla_label_generate_paper(ctx.handle, _stream(stream)), "polylla_label_generate_paper")


def label(ctx: Context, stream=None) -> None:
    _check(lib().polylla_label(ctx.handle, _stream(stream)), "polylla_label")


def generate(ctx: Context, stream=None) -> None:
    _check(lib().polylla_generate(ctx.handle, _stream(stream)), "polylla_generate")


def get_counts(ctx: Context, stream=None, check=True) -> dict:
    c = Counts()
    rc = lib().polylla_get_counts(ctx.handle, _stream(stream), ctypes.byref(c))
    if check:
        _check(rc, "polylla_get_counts")
    return c.as_dict()


def get_polygons(ctx: Context, offsets, loops, origin=None, twin=None, next=None, prev=None, stream=None):
    rc = lib().polylla_get_polygons(
        ctx.handle, _ptr(offsets), -1 if offsets is None else offsets.numel(), _ptr(loops),
        -1 if loops is None else loops.numel(), _ptr(origin), _ptr(twin), _ptr(next), _ptr(prev), _stream(stream))
    _check(rc, "polylla_get_polygons")


def get_triangle_polygons(ctx: Context, poly_of_tri: torch.Tensor, stream=None) -> None:
    """poly_of_tri (device int32 [T]) = index of the polygon containing each triangle;
    after get_polygons (it needs the polygon seeds)."""
    _check(lib().polylla_get_triangle_polygons(ctx.handle, _ptr(poly_of_tri), _stream(stream)),
           "polylla_get_triangle_polygons")


def get_triangle_regions(ctx: Context, region_of_tri: torch.Tensor, stream=None) -> None:
    """region_of_tri (device int32 [T]) = smallest triangle id of each triangle's
    terminal-edge region (the pre-repair Lepp partition); after label."""
    _check(lib().polylla_get_triangle_regions(ctx.handle, _ptr(region_of_tri), _stream(stream)),
           "polylla_get_triangle_regions")


def set_debug(ctx: Context, next_pre: torch.Tensor | None) -> None:
    _check(lib().polylla_set_debug(ctx.handle, _ptr(next_pre)), "polylla_set_debug")


def get_views(ctx: Context) -> dict:
    """Raw device pointers into the workspace, returned as torch tensor slices of it."""
    v = Views()
    _check(lib().polylla_get_views(ctx.handle, ctypes.byref(v)), "polylla_get_views")
    base = ctx.workspace.data_ptr()
    return {k: int(getattr(v, k)) - base for k, _ in Views._fields_}


def view_tensor(ctx: Context, offset: int, n: int, dtype) -> torch.Tensor:
    esz = torch.empty((), dtype=dtype).element_size()
    return ctx.workspace[offset:offset + n * esz].view(dtype)


def launch_count(ctx: Context) -> int:
    return int(lib().polylla_launch_count(ctx.handle))


def destroy(ctx: Context) -> None:
    if ctx.handle is not None and ctx.handle.value:
        lib().polylla_destroy(ctx.handle)
        ctx.handle = ctypes.c_void_p()


def profile_enable(on: bool = True) -> None:
    lib().polylla_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel group: (total ms, launches)} since the last read (synchronises)."""
    cap = 64
    names = (ctypes.c_char_p * cap)()
    ms = (ctypes.c_double * cap)()
    cnt = (ctypes.c_int64 * cap)()
    n = lib().polylla_profile_read(names, ms, cnt, cap)
    if n < 0:
        raise PolyllaError(-11, "polylla_profile_read")
    return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(n)}


def status_string(code: int) -> str:
    return lib().polylla_status_string(code).decode()


# ----------------------------------------------------------------------- conveniences

def run(xy: torch.Tensor, tri: torch.Tensor, stream=None, arrays=True, prev=False, debug=False,
        regions=False, check=False, paper=False, row_stride=0, sort=False) -> dict:
    """build -> label -> generate -> get_counts -> get_polygons on device tensors.
    Returns a dict of torch tensors (offsets, loops, seeds, [origin, twin, next, prev],
    [lcode, frontier0, frontier1, seed_bits, next_pre]) plus the counts."""
    V, T = xy.shape[0], tri.shape[0]
    ws = alloc_workspace(V, T, xy.device, row_stride=row_stride, sort=sort)
    ctx = build_halfedges(xy, tri, ws, stream, row_stride=row_stride, sort=sort)
    if check:
        check_manifold(ctx, stream)
    next_pre = None
    if debug:
        next_pre = torch.empty(6 * T, dtype=torch.int32, device=xy.device)
        set_debug(ctx, next_pre)
    if paper:
        label_generate_paper(ctx, stream)
    else:
        label(ctx, stream)
        generate(ctx, stream)
    counts = get_counts(ctx, stream)
    P, L, H = counts["n_polygons"], counts["n_loop_entries"], counts["n_halfedges"]
    dev = xy.device
    out = dict(counts)
    out.update(P=P, L=L, H=H)
    out["offsets"] = torch.empty(P + 1, dtype=torch.int32, device=dev)
    out["loops"] = torch.empty(max(L, 1), dtype=torch.int32, device=dev)
    kw = {}
    if arrays:
        for k in ("origin", "twin", "next"):
            out[k] = kw[k] = torch.empty(H, dtype=torch.int32, device=dev)
    if prev:
        out["prev"] = kw["prev"] = torch.empty(H, dtype=torch.int32, device=dev)
    get_polygons(ctx, out["offsets"], out["loops"], stream=stream, **kw)
    if regions:
        out["poly_of_tri"] = torch.empty(T, dtype=torch.int32, device=dev)
        get_triangle_polygons(ctx, out["poly_of_tri"], stream)
        out["region_of_tri"] = torch.empty(T, dtype=torch.int32, device=dev)
        get_triangle_regions(ctx, out["region_of_tri"], stream)
    c2 = get_counts(ctx, stream)  # synchronises; surfaces a capacity error
    out["loops"] = out["loops"][:L]
    v = get_views(ctx)
    nw = (3 * T + 31) // 32
    out["seeds"] = view_tensor(ctx, v["seeds"], P, torch.int32).clone()
    if debug:
        out["lcode"] = view_tensor(ctx, v["lcode"], T, torch.uint8).clone()
        for k in ("frontier0", "frontier1", "seed_bits"):
            out[k] = view_tensor(ctx, v[k], nw, torch.int32).clone()
        out["tips"] = view_tensor(ctx, v["tips"], counts["n_tips"], torch.int32).clone()
        out["next_pre"] = next_pre[:H].clone()
    out["launches"] = launch_count(ctx)
    assert c2["status"] == 0
    destroy(ctx)
    return out


def run_host(xy: np.ndarray, tri: np.ndarray, workspace: torch.Tensor | None = None, arrays=True, stream=None,
             pinned: dict | None = None) -> dict:
    """End to end from host numpy arrays through polylla_run_host (H2D, kernels, D2H)."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    V, T = xy.shape[0], tri.shape[0]
    if workspace is None:
        workspace = alloc_workspace(V, T)
    if pinned is None:
        pinned = alloc_host_outputs(T, arrays)
    c = Counts()
    a = {k: (None if pinned.get(k) is None else ctypes.c_void_p(pinned[k].data_ptr()))
         for k in ("offsets", "loops", "origin", "twin", "next")}
    rc = lib().polylla_run_host(
        ctypes.c_void_p(xy.ctypes.data), V, ctypes.c_void_p(tri.ctypes.data), T, _ptr(workspace),
        workspace.numel(), a["offsets"], pinned["offsets"].numel(), a["loops"], pinned["loops"].numel(),
        a["origin"], a["twin"], a["next"], 6 * T, ctypes.byref(c), _stream(stream))
    _check(rc, "polylla_run_host")
    d = c.as_dict()
    P, L, H = d["n_polygons"], d["n_loop_entries"], d["n_halfedges"]
    out = dict(d)
    out.update(P=P, L=L, H=H, offsets=pinned["offsets"][:P + 1], loops=pinned["loops"][:L])
    if arrays:
        for k in ("origin", "twin", "next"):
            out[k] = pinned[k][:H]
    return out


def alloc_host_outputs(T: int, arrays=True, pin=True) -> dict:
    mk = (lambda n: torch.empty(n, dtype=torch.int32, pin_memory=pin))
    d = dict(offsets=mk(T + 1), loops=mk(3 * T))
    if arrays:
        for k in ("origin", "twin", "next"):
            d[k] = mk(6 * T)
    return d


class GraphStep:
    """One whole conversion (build -> label -> generate -> CSR) captured as a CUDA graph on
    a fixed workspace/inputs/outputs and replayed with a single launch: the ~20 kernel
    launches of a step become one graph launch (the small configs are launch-bound).
    The C ABI is called unchanged during capture; its kernels read the mesh size from the
    workspace counters on the device, so a replay recomputes everything."""

    def __init__(self, xy, tri, workspace, offsets, loops, stream=None, paper=False, row_stride=0, sort=False):
        self.stream = stream or torch.cuda.Stream(device=xy.device)

        def lg(ctx, st):
            if paper:
                label_generate_paper(ctx, st)
            else:
                label(ctx, st)
                generate(ctx, st)
        self.args = (xy, tri, workspace, offsets, loops)
        # warm once outside capture (lazy CUDA attribute setup inside the library)
        with torch.cuda.stream(self.stream):
            ctx = build_halfedges(xy, tri, workspace, self.stream, row_stride=row_stride, sort=sort)
            lg(ctx, self.stream)
            get_polygons(ctx, offsets, loops, stream=self.stream)
            self.launches = launch_count(ctx)
            destroy(ctx)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            s = torch.cuda.current_stream()
            ctx = build_halfedges(xy, tri, workspace, s, row_stride=row_stride, sort=sort)
            lg(ctx, s)
            get_polygons(ctx, offsets, loops, stream=s)
            destroy(ctx)

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()


class HostPipeline:
    """End-to-end conversion of a stream of meshes from pinned HOST buffers to pinned HOST
    results, three-stage pipelined (the copies are ~90% of the
    end-to-end time and PCIe is full duplex):

        up stream      H2D(xy_i, tri_i) ----------> H2D(xy_{i+1}, ...)
        compute stream           build/label/generate/CSR(i)      CSR(i+1) ...
        down stream                                      D2H(CSR_i, origin/twin/next_i)
                                                         (overlaps H2D(i+1))

    Two slots (workspace + device inputs + CSR staging) alternate; CUDA events order the
    reuse of a slot.  Every step still moves its own inputs up and its own results down
    through the C ABI (polylla_build_halfedges ... polylla_get_polygons + async copies);
    the one host sync per mesh is polylla_get_counts (it sizes the D2H copies)."""

    def __init__(self, n_vertices: int, n_triangles: int, arrays: bool = True, device="cuda"):
        self.V, self.T, self.arrays = n_vertices, n_triangles, arrays
        dev = torch.device(device)
        self.up, self.comp, self.down = (torch.cuda.Stream(device=dev) for _ in range(3))
        self.slots = []
        for _ in range(2):
            self.slots.append(dict(
                ws=alloc_workspace(n_vertices, n_triangles, dev),
                xy=torch.empty((n_vertices, 2), dtype=torch.float64, device=dev),
                tri=torch.empty((n_triangles, 3), dtype=torch.int32, device=dev),
                offsets=torch.empty(n_triangles + 1, dtype=torch.int32, device=dev),
                loops=torch.empty(3 * n_triangles, dtype=torch.int32, device=dev),
                ev_up=torch.cuda.Event(), ev_comp=torch.cuda.Event(), ev_down=torch.cuda.Event(),
                used=False))

    def run(self, inputs, outputs):
        """inputs: list of (xy_pinned [V,2] f64, tri_pinned [T,3] i32) host tensors;
        outputs: list of dicts of pinned host tensors (offsets [T+1], loops [3T], and
        origin/twin/next [6T] when arrays=True).  Returns the per-mesh counts; the results
        are complete in `outputs` when this returns."""
        counts = [None] * len(inputs)
        pending = None  # (index, slot, ctx) waiting for its D2H

        def drain(item):
            i, sl, ctx = item
            c = get_counts(ctx, self.comp)  # the one host sync of mesh i (compute stream)
            counts[i] = c
            P, L, H = c["n_polygons"], c["n_loop_entries"], c["n_halfedges"]
            o = outputs[i]
            with torch.cuda.stream(self.down):
                self.down.wait_event(sl["ev_comp"])
                o["offsets"][:P + 1].copy_(sl["offsets"][:P + 1], non_blocking=True)
                o["loops"][:L].copy_(sl["loops"][:L], non_blocking=True)
                if self.arrays:
                    v = get_views(ctx)
                    for k in ("origin", "twin", "next"):
                        o[k][:H].copy_(view_tensor(ctx, v[k], H, torch.int32), non_blocking=True)
                sl["ev_down"].record(self.down)
            destroy(ctx)

        for i, (xy_h, tri_h) in enumerate(inputs):
            sl = self.slots[i % 2]
            V, T = xy_h.shape[0], tri_h.shape[0]
            with torch.cuda.stream(self.up):
                if sl["used"]:
                    self.up.wait_event(sl["ev_comp"])  # the previous mesh of this slot read its inputs
                sl["xy"][:V].copy_(xy_h, non_blocking=True)
                sl["tri"][:T].copy_(tri_h, non_blocking=True)
                sl["ev_up"].record(self.up)
            # drain mesh i-1 before mesh i's kernels are queued: its counts sync waits for
            # its own kernels only, and its D2H then runs while H2D(i) is in flight
            if pending is not None:
                drain(pending)
                pending = None
            self.comp.wait_event(sl["ev_up"])
            if sl["used"]:
                self.comp.wait_event(sl["ev_down"])  # its workspace was downloaded
            ctx = build_halfedges(sl["xy"][:V], sl["tri"][:T], sl["ws"], self.comp)
            label(ctx, self.comp)
            generate(ctx, self.comp)
            get_polygons(ctx, sl["offsets"], sl["loops"], stream=self.comp)
            sl["ev_comp"].record(self.comp)
            sl["used"] = True
            pending = (i, sl, ctx)
        if pending is not None:
            drain(pending)
        self.down.synchronize()
        return counts
