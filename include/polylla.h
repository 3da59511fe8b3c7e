/*
 * polylla.h -- C ABI of libpolylla.so, a B200-native (sm_100a) implementation of the
 * data-parallel core of Polylla as GPolylla defines it (arXiv 2403.14723, PAPER.md).
 *
 * Problem statement: a triangulation tau = (V, E) -- vertex
 * coordinates plus a triangle index list -- is converted into a polygonal mesh
 * tau' = (V, E') represented by the SAME half-edge array with rewired next links
 * ("unlink instead of delete"), plus one seed half-edge per
 * polygon from which each polygon is rebuilt.  Every step runs in
 * hand-written CUDA kernels; the host code below only validates arguments, carves
 * the caller's workspace and launches kernels.
 *
 * Conventions (readings R1-R18):
 *   - indices are 0-based; vertex ids (tri, origin, loops) are int32 (V <= 2^31 - 1);
 *     half-edge ids (twin, next, prev, seeds) and CSR offsets are UNSIGNED 32-bit, so
 *     a mesh may have up to H = 2^32 - 2 half-edges (the capacity question of PAPER.md
 *     L55: twice the int32 ceiling).  For H <= 2^31 - 1 the
 *     arrays read identically as int32 (the int32 reading of every earlier version);
 *   - coordinates are float64 interleaved (x0,y0,x1,y1,...) = a contiguous
 *     torch.float64 tensor [V,2];
 *   - interior half-edge e = 3f+k has origin tri'[f][k] and target tri'[f][(k+1)%3],
 *     where tri' is the input triangle re-oriented CCW (a CW triangle has its 2nd and
 *     3rd vertex swapped, R10); next_in(e) = 3f+(k+1)%3;
 *   - border half-edges get ids 3T + rank(e) over the unmatched interior half-edges e
 *     in ascending order (R9), origin(b) = target(e), and next(b) chains the
 *     exterior face;
 *   - H = 3T + B half-edges in total.
 *
 * Pointers: unless stated otherwise every array pointer is a CUDA DEVICE pointer
 * (cudaMalloc'ed or a torch CUDA tensor's data_ptr()).  `stream` is a cudaStream_t
 * (NULL = the legacy default stream).  Calls are asynchronous on `stream` except
 * polylla_get_counts and polylla_run_host, which synchronise it.
 *
 * Ownership: the caller owns xy, tri, the workspace and every output buffer; they
 * must stay alive until polylla_destroy.  The library never calls cudaMalloc and
 * never writes xy or tri.  A ctx is a small host struct (malloc'ed by
 * polylla_build_halfedges, freed by polylla_destroy) used by one stream / one host
 * thread at a time.
 *
 * Errors: argument errors are returned synchronously.  Errors found on the device
 * (bad input mesh, walk bounds) are OR-ed into a device status word and returned
 * by the next synchronising call (polylla_get_counts / polylla_run_host); once set,
 * later kernels of the same ctx return immediately.
 *
 * Call order: build -> label -> generate -> get_counts -> get_polygons; get_views
 * after build.  Out-of-order calls return POLYLLA_E_CALL_ORDER.
 */
#ifndef POLYLLA_H
#define POLYLLA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define POLYLLA_API __attribute__((visibility("default")))
#else
#define POLYLLA_API
#endif

typedef struct polylla_ctx polylla_ctx;
typedef void* polylla_stream; /* cudaStream_t */

typedef enum {
  POLYLLA_OK = 0,
  POLYLLA_E_INVALID_ARGUMENT = -1,    /* null/misaligned pointer, V < 3, T < 1 */
  POLYLLA_E_DANGLING_INDEX = -2,      /* a triangle index outside [0, V) */
  POLYLLA_E_DEGENERATE_TRI = -3,      /* zero signed area or repeated vertex */
  POLYLLA_E_NON_MANIFOLD_EDGE = -4,   /* an edge in > 2 triangles, or twice in one direction */
  POLYLLA_E_NON_MANIFOLD_VERTEX = -5, /* a vertex with > 1 outgoing border half-edge (border chain ambiguous) */
  POLYLLA_E_INDEX_OVERFLOW = -6,      /* 3T + max_border > 2^32 - 2, or V > INT32_MAX */
  POLYLLA_E_WORKSPACE = -7,           /* workspace too small or not 256-byte aligned; or (device) B > max_border */
  POLYLLA_E_WALK_BOUND = -8,          /* SPEC.md L160/L174/L260: a rotation or loop walk did not close */
  POLYLLA_E_UNSEEDED_LOOP = -9,       /* sum of loop lengths != #interior frontier half-edges (exact-tie Lepp cycle, R12) */
  POLYLLA_E_CALL_ORDER = -10,
  POLYLLA_E_CUDA = -11,               /* a CUDA runtime call failed */
  POLYLLA_E_CAPACITY = -12            /* an output buffer passed to get_polygons is too small */
} polylla_status;

/* Counts of one conversion (returned by polylla_get_counts / polylla_run_host). */
typedef struct {
  int64_t n_vertices;      /* V */
  int64_t n_triangles;     /* T */
  int64_t n_halfedges;     /* H = 3T + B */
  int64_t n_border;        /* B */
  int64_t n_polygons;      /* P: output polygons (after repair) */
  int64_t n_loop_entries;  /* L: CSR loop entries = #interior frontier half-edges */
  int64_t n_tips;          /* barrier tips repaired */
  int64_t n_flips;         /* CW input triangles re-oriented */
  int64_t n_leftover;      /* half-edges whose twin was matched outside their build tile */
  int64_t n_deferred;      /* half-edges whose label/rewire needed data outside their tile (polylla_label) */
  int64_t n_seed_deferred; /* seeds walked globally: polygon not closed inside the build tile, or a repair half */
  int32_t status;          /* the device status, as a polylla_status */
  int32_t reserved;
} polylla_counts;

/* Bytes of device workspace needed for a mesh with V vertices and T triangles
 * (worst case B = 3T; includes staging for polylla_run_host).  Host-only. */
POLYLLA_API size_t polylla_workspace_bytes(int64_t n_vertices, int64_t n_triangles);

/* Workspace / build flags. */
#define POLYLLA_WS_STAGING 1u /* hold the host-buffer staging regions of polylla_run_host */
#define POLYLLA_BUILD_SORT 2u /* build tiles over triangles ordered by the Morton cell of their centroid
                                 (any input order; ignores row_stride): a performance option, same results */

/* Bytes of device workspace for a mesh with at most max_border border half-edges
 * (0 <= max_border <= 3T; e.g. 4(s-1) for an s x s grid), with POLYLLA_WS_STAGING in
 * flags run_host's staging, and a row stride hint (0: none; see
 * polylla_build_halfedges_ex).  polylla_workspace_bytes(V, T) ==
 * polylla_workspace_bytes_ex(V, T, 3T, POLYLLA_WS_STAGING, 0).  The origin/twin/next
 * regions shrink from 6T to 3T + max_border entries and the staging (12T + 12T + 16V
 * bytes) is dropped: the capacity path for meshes near the HBM limit (SURVEY.md §8(f)
 * NEXT-3).  Returns 0 on invalid arguments.  Host-only. */
POLYLLA_API size_t polylla_workspace_bytes_ex(int64_t n_vertices, int64_t n_triangles, int64_t max_border,
                                              uint32_t flags, int64_t row_stride);

/* Half-edge construction (SPEC.md L45-53 build_from_triangles),
 * moved on-device, fused with the longest-edge labelling of Alg. 2 / Alg. 7
 * (PAPER.md L351-376, L608-635):
 *   xy  [V][2] float64, 16-byte aligned;  tri [T][3] int32, 4-byte aligned;
 *   workspace: >= polylla_workspace_bytes(V, T) bytes, 256-byte aligned.
 * Orients triangles CCW, writes origin[], pairs twins (tile-local shared-memory
 * hash + global fallback), creates and chains border half-edges, computes each
 * triangle's longest edge (first maximum of the FP64 squared lengths of its
 * half-edges 3f, 3f+1, 3f+2; no FMA contraction).  Asynchronous; *ctx_out receives
 * a new context on success. */
POLYLLA_API polylla_status polylla_build_halfedges(const double* xy, int64_t n_vertices, const int32_t* tri,
                                                   int64_t n_triangles, void* workspace, size_t workspace_bytes,
                                                   polylla_stream stream, polylla_ctx** ctx_out);

/* polylla_build_halfedges over a workspace laid out by polylla_workspace_bytes_ex with
 * the same max_border, flags and row_stride (the layout must match).  A mesh with more
 * than max_border border half-edges sets POLYLLA_E_WORKSPACE in the device status
 * (returned by polylla_get_counts); nothing is written past the bound.
 * row_stride: 0, or R > 0 when the triangle list is row-major with rows of R triangles
 * (R divides T; e.g. R = 2(s-1) for the Alg. 13 grids): the build then
 * tiles 16-row x 128-triangle patches instead of 2,048 consecutive triangles, so a tile
 * cuts ~3% of its edges instead of a third (a performance hint only: the results are the
 * same bits for any R; an R that does not divide T is ignored).
 * polylla_build_halfedges(...) == polylla_build_halfedges_ex(..., 3T, POLYLLA_WS_STAGING, 0, ...). */
POLYLLA_API polylla_status polylla_build_halfedges_ex(const double* xy, int64_t n_vertices, const int32_t* tri,
                                                      int64_t n_triangles, int64_t max_border, uint32_t flags,
                                                      int64_t row_stride, void* workspace, size_t workspace_bytes,
                                                      polylla_stream stream, polylla_ctx** ctx_out);

/* Exact non-manifold-edge check (SPEC.md L49 NonManifoldEdge), opt-in.  The build
 * detects an edge in more than two triangles (or twice in one direction) when all of
 * its copies fall in one 2,048-triangle build tile or all of them cross tiles; a copy
 * that pairs inside its tile while a further copy lies in another tile is seen only by
 * this pass (R20).  Every interior half-edge looks its undirected key up in a
 * global hash (dead workspace scratch); a second copy in the same direction, or a third
 * copy, ORs POLYLLA_E_NON_MANIFOLD_EDGE into the device status (returned by the next
 * polylla_get_counts).  Call after polylla_build_halfedges and before
 * polylla_get_triangle_polygons / a host-pointer prev (which reuse the same scratch);
 * asynchronous (2 launches).  Needs 3T + max_border <= INT32_MAX (else
 * POLYLLA_E_INDEX_OVERFLOW): its slots carry a flag bit next to the half-edge id. */
POLYLLA_API polylla_status polylla_check_manifold(polylla_ctx* ctx, polylla_stream stream);

/* Label phase (Alg. 8-9): frontier bits F[e] = border(e) or
 * border(twin e) or (not L[e] and not L[twin e]); seed bits for terminal and
 * terminal-border edges on the smaller interior half-edge.  Fused with the unlink
 * rewire (Alg. 11, read per R1/R3/R14): every interior frontier
 * half-edge e gets next[e] = the first frontier half-edge met rotating about
 * target(e) from next_in(e); non-frontier interior half-edges keep next_in; barrier
 * tips are detected as next[e] == twin[e] (R4).  Asynchronous. */
POLYLLA_API polylla_status polylla_label(polylla_ctx* ctx, polylla_stream stream);

/* Generate (Alg. 10, 12, Overwrite seeds, Scan): repair every
 * barrier tip (middle edge = floor((deg-1)/2) rotations past its frontier edge,
 * R5, snapshot R6) and re-rewire around the touched vertices; land every seed on
 * its polygon, walk the polygon, keep its minimum half-edge id as the canonical
 * seed; compact canonical seeds in ascending order and scan the
 * loop lengths into CSR offsets.  Asynchronous. */
POLYLLA_API polylla_status polylla_generate(polylla_ctx* ctx, polylla_stream stream);

/* Ablation: label + generate by the paper's own GPU kernel
 * sequence instead of polylla_label + polylla_generate -- LLK (Alg. 7, per triangle),
 * LFK (Alg. 8) and LSK (Alg. 9, per half-edge), LEK (Alg. 10: every VERTEX counts its
 * frontier edges; barrier tips get their middle edge before the rewire), CaK (Alg. 11:
 * next and prev of every frontier half-edge by rotation), SFK (Alg. 12) and Overwrite
 * seeds (per seed), then Scan and compact, one thread per element.
 * Same results as the default path, bit for bit.  Call after polylla_build_halfedges
 * (stage 1); afterwards get_counts / get_polygons as usual (get_triangle_polygons and
 * get_triangle_regions too).  Asynchronous (~14 launches and memsets).  Needs
 * 3T + max_border <= INT32_MAX (else POLYLLA_E_INDEX_OVERFLOW). */
POLYLLA_API polylla_status polylla_label_generate_paper(polylla_ctx* ctx, polylla_stream stream);

/* Synchronises `stream` and returns the counts and the device status.  The return
 * value is counts->status (POLYLLA_OK when the conversion succeeded). */
POLYLLA_API polylla_status polylla_get_counts(polylla_ctx* ctx, polylla_stream stream, polylla_counts* counts);

/* Polygon extraction (moved on-device).  offsets [P+1] and loops [L]
 * are device pointers with capacities offsets_cap >= P+1 and loops_cap >= L
 * (P <= T and L <= 3T always hold, so T+1 and 3T are safe without a sync):
 * polygon p is loops[offsets[p] .. offsets[p+1]) = origin[x0], origin[x1], ... with
 * x0 = seeds[p] (ascending canonical seeds) and x_{i+1} = next[x_i].  origin, twin,
 * next, prev: optional [H] outputs (NULL to skip; device or host pointers; copied
 * with cudaMemcpyAsync -- origin/twin/next and a host prev need polylla_get_counts
 * first, for H).  prev is the inverse of next on frontier and border half-edges and
 * prev_in elsewhere; it is built on the device (into the caller's array when that is
 * device memory, else into workspace scratch that is then copied out).  offsets and
 * loops are both given or both NULL.  Asynchronous; a too-small capacity sets
 * POLYLLA_E_CAPACITY in the device status. */
POLYLLA_API polylla_status polylla_get_polygons(polylla_ctx* ctx, uint32_t* offsets, int64_t offsets_cap,
                                                int32_t* loops, int64_t loops_cap, int32_t* origin, uint32_t* twin,
                                                uint32_t* next, uint32_t* prev, polylla_stream stream);

/* Per-triangle polygon ids (the output polygons as unions of triangles: the terminal-edge
 * regions of PAPER.md L76-L128 after the barrier repair):
 *   poly_of_tri[t] = the index, in polylla_get_polygons' order, of the polygon whose loop
 *   bounds the piece of t -- the triangles connected to t across non-frontier (F1 = 0)
 *   edges; where several loops bound one piece (around a hole of the mesh), the smallest.
 * poly_of_tri: device int32 [T], written by the caller-owned pointer; -1 is never written
 * for a valid conversion.  Needs a previous polylla_get_polygons with offsets/loops on this
 * ctx (it reads the polygon seeds; same stream, or synchronise), else E_CALL_ORDER.  The
 * ids are valid only if a later polylla_get_counts returns POLYLLA_OK: when the device
 * status is set (e.g. a capacity error in get_polygons, so no seeds were written) every
 * entry is -1.  Uses dead workspace scratch; asynchronous (4 launches). */
POLYLLA_API polylla_status polylla_get_triangle_polygons(polylla_ctx* ctx, int32_t* poly_of_tri, polylla_stream stream);

/* Per-triangle terminal-edge-region ids (the pre-repair Lepp
 * partition): the terminal-edge regions of PAPER.md Defs. 1-2 (L121-128) -- the triangles
 * whose longest-edge propagating paths end at the same terminal edge -- which the
 * data-parallel Lepp refinement of PAPER.md L76 works on, and which the repair (L517-570)
 * later splits into the output polygons.  On the device a region is the piece of
 * triangles connected across interior non-frontier edges of the label-phase frontier F0:
 *   region_of_tri[t] = the smallest triangle index of t's region.
 * region_of_tri: device int32 [T], caller-owned.  Call after polylla_label (stage >= 2);
 * valid only if a later polylla_get_counts returns POLYLLA_OK (else every entry is -1).
 * Uses dead workspace scratch (shared with get_triangle_polygons, check_manifold and a
 * host-pointer prev: not concurrently); asynchronous (3 launches). */
POLYLLA_API polylla_status polylla_get_triangle_regions(polylla_ctx* ctx, int32_t* region_of_tri,
                                                        polylla_stream stream);

/* Device views into the workspace (valid until polylla_destroy / workspace reuse).
 * Any pointer argument may be NULL.  Sizes: origin/twin/next [H]; lcode [T] (k* of
 * each triangle); frontier0 / frontier1 / seed_bits: bit-vectors of uint32 words
 * over the interior half-edges [0, 3T) (bit e%32 of word e/32; border half-edges
 * are frontier by definition); seeds [P] (canonical seed of each polygon, written by
 * polylla_get_polygons). */
typedef struct {
  const int32_t* origin;
  const uint32_t* twin;
  const uint32_t* next;
  const uint8_t* lcode;
  const uint32_t* frontier0;
  const uint32_t* frontier1;
  const uint32_t* seed_bits;
  const uint32_t* seeds;
  const uint32_t* tips;  /* [n_tips] incoming frontier half-edge of each barrier tip (unordered) */
} polylla_views;
POLYLLA_API polylla_status polylla_get_views(polylla_ctx* ctx, polylla_views* views);

/* Debug: when next_pre (device [H]) is non-NULL, polylla_generate first copies the
 * pre-repair next array into it (stage-wise parity tests). */
POLYLLA_API polylla_status polylla_set_debug(polylla_ctx* ctx, uint32_t* next_pre);

/* End to end from HOST buffers (pageable or pinned): H2D of xy/tri into the
 * workspace, build -> label -> generate, one sync, extraction, D2H of the CSR
 * (offsets [P+1], loops [L]) and, if non-NULL, origin/twin/next [H] -- all on
 * `stream`, synchronised before returning.  Host capacities as in get_polygons
 * (origin/twin/next need n_halfedges <= 6T entries).  *counts receives the counts.
 * The workspace is laid out by polylla_workspace_bytes (staging included).  The ctx is
 * destroyed before returning. */
POLYLLA_API polylla_status polylla_run_host(const double* xy_host, int64_t n_vertices, const int32_t* tri_host,
                                            int64_t n_triangles, void* workspace, size_t workspace_bytes,
                                            uint32_t* offsets_host, int64_t offsets_cap, int32_t* loops_host,
                                            int64_t loops_cap, int32_t* origin_host, uint32_t* twin_host,
                                            uint32_t* next_host, int64_t halfedge_cap, polylla_counts* counts,
                                            polylla_stream stream);

POLYLLA_API void polylla_destroy(polylla_ctx* ctx);

/* Optional per-kernel timing (process-wide, host-only state): when enabled, CUDA
 * events are recorded on the launching stream around each kernel group
 * (k_build_tile, k_left_match, k_border_scan, k_border_next, k_label_rewire,
 * k_repair, k_seed_walk, k_canon_scan, k_extract).  polylla_profile_read
 * synchronises on the recorded events, writes up to `cap` (name, total ms, launch
 * count) triples accumulated since the last read/enable, clears them and returns
 * the number written (< 0 on a CUDA error).  Names are valid until the next read. */
POLYLLA_API void polylla_profile_enable(int on);
POLYLLA_API int polylla_profile_read(const char** names, double* total_ms, int64_t* count, int cap);
POLYLLA_API const char* polylla_status_string(polylla_status s);

/* Number of kernel launches issued by the calls since the ctx was built (for the
 * bench's gpu_launches claim). */
POLYLLA_API int64_t polylla_launch_count(const polylla_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* POLYLLA_H */
