// capi.cu -- the C ABI of libpolylla.so (include/polylla.h): argument validation,
// workspace carving, call-order state, kernel orchestration.  No compute here: every
// step of the conversion runs in the kernels of build.cu / label.cu / generate.cu /
// extract.cu.
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "internal.cuh"

namespace polylla {

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static int64_t hash_cap_max_for(int64_t T) {
  int64_t c = 1024;
  while (c < 2 * 3 * T && c < (int64_t(1) << 31)) c <<= 1;
  return c;
}

struct Layout {
  size_t off[48];
  size_t total;
};

// region order; sizes in bytes.  Hmax = 3T + Bmax (the caller's bound on the border
// half-edges; 3T covers every mesh); the run_host staging regions only when `staging`.
static Layout layout(int64_t V, int64_t T, int64_t Bmax, bool staging, int64_t R, bool sorted) {
  const int64_t Hmax = 3 * T + Bmax;
  const Tiling tg = make_tiling(T, R, sorted);
  const int64_t bt = tg.ntiles;  // build tiles (grid tilings have more, partial ones)
  const bool scat = tg.mode != kTileContig;
  const int64_t ct = (T + 2047) / 2048;          // contiguous tiles (emission, canonical sums)
  const int64_t nw = (3 * T + 31) / 32;
  const int64_t nb = (nw + 2047) / 2048 + 1;
  const int64_t cap = hash_cap_max_for(T);
  const size_t sz[] = {
      (size_t)Hmax * 4,       // 0 origin
      (size_t)Hmax * 4,       // 1 twin
      (size_t)Hmax * 4,       // 2 next
      (size_t)T,              // 3 lcode
      (size_t)nw * 4,         // 4 F0
      (size_t)nw * 4,         // 5 F1
      (size_t)nw * 4,         // 6 S
      (size_t)nw * 4,         // 7 TB: barrier tips (F0, F1, S, TB equally spaced: k_tile stores them by offset)
      (size_t)((bt > ct ? bt : ct) + 1) * 4,  // 8 per-tile (or per-chunk) border counts / bases
      (size_t)(3 * T),        // 9 len (bytes)
      (size_t)(3 * T) * 8,    // 10 left_key
      (size_t)(3 * T) * 4,    // 11 left_e
      (size_t)cap * 4,        // 12 ehash
      (size_t)V * 4,          // 13 vmap
      0,                      // 14 (unused)
      (size_t)V * 4,          // 15 tips
      (size_t)(2 * V) * 4,    // 16 aff
      scat ? (size_t)nw * 4 : 0,  // 17 BB: unmatched leftovers (grid / sorted tiling)
      (size_t)nb * 8,         // 18 scan_a
      (size_t)nb * 8,         // 19 scan_b
      (size_t)nb * 8,         // 20 scan_c
      (size_t)T * 4,          // 21 seeds
      (size_t)(T + 1) * 4,    // 22 offsets
      staging ? (size_t)(3 * T) * 4 : 0,  // 23 loops staging (run_host)
      staging ? (size_t)(2 * V) * 8 : 0,  // 24 xy staging
      staging ? (size_t)(3 * T) * 4 : 0,  // 25 tri staging
      sizeof(DevCounters),    // 26 counters
      (size_t)(3 * T) * 4,    // 27 deferred half-edges
      (size_t)nw * 4,         // 28 SDB: seeds for the global seed walk
      (size_t)nw * 4,         // 29 per-word loop lengths
      (size_t)nw * 4,         // 30 C
      (size_t)(2 * bt + 2) * 4,  // 31 per-build-tile leftover / deferred counts
      (size_t)(3 * ((T + 2047) / 2048) + 2) * 4,  // 32 per-tile canonical-seed sums
      (size_t)(2 * ((T + 2047) / 2048) + 2) * 4,  // 33 per-tile polygon / loop-entry bases
      sorted ? (size_t)T * 4 : 0,                 // 34 (sorted tiling) perm
      sorted ? (size_t)T * 4 : 0,                 // 35 (sorted tiling) Morton cell keys
      sorted ? (size_t)kSortCells * 4 : 0,        // 36 (sorted tiling) cell counts / cursors
      sorted ? (size_t)32 : 0,                    // 37 (sorted tiling) bounding box
  };
  Layout L{};
  static_assert(sizeof(sz) / sizeof(sz[0]) <= sizeof(L.off) / sizeof(L.off[0]), "Layout::off too small");
  size_t o = 0;
  for (size_t i = 0; i < sizeof(sz) / sizeof(sz[0]); ++i) {
    L.off[i] = o;
    o += align_up(sz[i]);
  }
  L.total = o;
  return L;
}

size_t workspace_bytes(int64_t V, int64_t T, int64_t Bmax, bool staging, int64_t R, bool sorted) {
  return layout(V, T, Bmax, staging, R, sorted).total;
}

bool carve(Ctx* c, void* ws, size_t bytes) {
  const bool sorted = c->tiling.mode == kTileSorted;  // (new_ctx: the requested tiling)
  c->tiling = make_tiling(c->T, c->tiling.R, sorted);
  const Layout L = layout(c->V, c->T, c->Bmax, c->staging, c->tiling.R, sorted);
  if (bytes < L.total || (reinterpret_cast<uintptr_t>(ws) & 255)) return false;
  char* b = static_cast<char*>(ws);
  c->Hmax = 3 * c->T + c->Bmax;
  c->origin = reinterpret_cast<int32_t*>(b + L.off[0]);
  c->twin = reinterpret_cast<hid*>(b + L.off[1]);
  c->next = reinterpret_cast<hid*>(b + L.off[2]);
  c->lcode = reinterpret_cast<uint8_t*>(b + L.off[3]);
  c->F0 = reinterpret_cast<uint32_t*>(b + L.off[4]);
  c->F1 = reinterpret_cast<uint32_t*>(b + L.off[5]);
  c->S = reinterpret_cast<uint32_t*>(b + L.off[6]);
  c->TB = reinterpret_cast<uint32_t*>(b + L.off[7]);
  c->bcnt = reinterpret_cast<uint32_t*>(b + L.off[8]);
  c->len = reinterpret_cast<uint8_t*>(b + L.off[9]);
  c->left_key = reinterpret_cast<unsigned long long*>(b + L.off[10]);
  c->left_e = reinterpret_cast<hid*>(b + L.off[11]);
  c->ehash = b + L.off[12];
  c->vmap = reinterpret_cast<hid*>(b + L.off[13]);
  c->hash_cap_max = hash_cap_max_for(c->T);
  c->tips = reinterpret_cast<hid*>(b + L.off[15]);
  c->aff = reinterpret_cast<hid*>(b + L.off[16]);
  c->mids = nullptr;
  c->BB = c->tiling.mode != kTileContig ? reinterpret_cast<uint32_t*>(b + L.off[17]) : nullptr;
  if (sorted) {
    c->tiling.perm = reinterpret_cast<int32_t*>(b + L.off[34]);
    c->sort_key = reinterpret_cast<uint32_t*>(b + L.off[35]);
    c->sort_hist = reinterpret_cast<uint32_t*>(b + L.off[36]);
    c->sort_bbox = reinterpret_cast<unsigned long long*>(b + L.off[37]);
  }
  c->scan_a = reinterpret_cast<long long*>(b + L.off[18]);
  c->scan_b = reinterpret_cast<long long*>(b + L.off[19]);
  c->scan_c = reinterpret_cast<long long*>(b + L.off[20]);
  c->seeds = reinterpret_cast<hid*>(b + L.off[21]);
  c->offsets = reinterpret_cast<uint32_t*>(b + L.off[22]);
  c->loops = c->staging ? reinterpret_cast<int32_t*>(b + L.off[23]) : nullptr;
  c->xy_stage = c->staging ? reinterpret_cast<double*>(b + L.off[24]) : nullptr;
  c->tri_stage = c->staging ? reinterpret_cast<int32_t*>(b + L.off[25]) : nullptr;
  c->ctr = reinterpret_cast<DevCounters*>(b + L.off[26]);
  c->def_e = reinterpret_cast<hid*>(b + L.off[27]);
  c->SDB = reinterpret_cast<uint32_t*>(b + L.off[28]);
  c->C = reinterpret_cast<uint32_t*>(b + L.off[30]);
  c->cnt_ld = reinterpret_cast<int32_t*>(b + L.off[31]);
  c->tsum = reinterpret_cast<int32_t*>(b + L.off[32]);
  c->tbase = reinterpret_cast<uint32_t*>(b + L.off[33]);
  c->wlen = reinterpret_cast<int32_t*>(b + L.off[29]);
  c->n_words = (3 * c->T + 31) / 32;
  return true;
}

static polylla_status map_status(uint32_t st) {
  if (!st) return POLYLLA_OK;
  if (st & ST_DANGLING) return POLYLLA_E_DANGLING_INDEX;
  if (st & ST_DEGENERATE) return POLYLLA_E_DEGENERATE_TRI;
  if (st & ST_NONMANIFOLD_EDGE) return POLYLLA_E_NON_MANIFOLD_EDGE;
  if (st & ST_NONMANIFOLD_VERTEX) return POLYLLA_E_NON_MANIFOLD_VERTEX;
  if (st & ST_OVERFLOW) return POLYLLA_E_INDEX_OVERFLOW;
  if (st & ST_WALK) return POLYLLA_E_WALK_BOUND;
  if (st & ST_UNSEEDED) return POLYLLA_E_UNSEEDED_LOOP;
  if (st & ST_CAPACITY) return POLYLLA_E_CAPACITY;
  return POLYLLA_E_WORKSPACE;  // (ST_BORDER_CAP: B above the workspace's border bound; ST_INTERNAL)
}

// ------------------------------------------------------------------ profiling
struct ProfEntry {
  const char* name;
  cudaEvent_t a, b;
};
static bool g_prof = false;
static std::vector<cudaEvent_t> g_pool;
static size_t g_pool_used = 0;
static std::vector<ProfEntry> g_entries;
static const char* g_open = nullptr;
static cudaEvent_t g_open_ev;

static cudaEvent_t prof_event() {
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_pool.push_back(e);
  }
  return g_pool[g_pool_used++];
}

void prof_mark(cudaStream_t s, const char* name) {
  if (!g_prof) return;
  cudaEvent_t e = prof_event();
  cudaEventRecord(e, s);
  if (g_open) g_entries.push_back({g_open, g_open_ev, e});
  g_open = name;
  g_open_ev = e;
}

void prof_end(cudaStream_t s) {
  if (!g_prof || !g_open) return;
  cudaEvent_t e = prof_event();
  cudaEventRecord(e, s);
  g_entries.push_back({g_open, g_open_ev, e});
  g_open = nullptr;
}

}  // namespace polylla

using namespace polylla;

struct polylla_ctx {
  Ctx c;
};

static inline cudaStream_t S(polylla_stream s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

POLYLLA_API size_t polylla_workspace_bytes(int64_t n_vertices, int64_t n_triangles) {
  if (n_vertices < 0 || n_triangles < 0) return 0;
  return workspace_bytes(n_vertices, n_triangles, 3 * n_triangles, true);
}

POLYLLA_API size_t polylla_workspace_bytes_ex(int64_t n_vertices, int64_t n_triangles, int64_t max_border,
                                              uint32_t flags, int64_t row_stride) {
  if (n_vertices < 0 || n_triangles < 0 || max_border < 0 || max_border > 3 * n_triangles || row_stride < 0) return 0;
  return workspace_bytes(n_vertices, n_triangles, max_border, (flags & POLYLLA_WS_STAGING) != 0, row_stride,
                         (flags & POLYLLA_BUILD_SORT) != 0);
}

// index limits (NEXT-3): vertex ids int32; half-edge ids uint32 with H <= 2^32 - 2
static bool index_ok(int64_t V, int64_t T, int64_t Bmax) {
  return V <= 0x7fffffffLL && 3 * T + Bmax <= kMaxHalfedges;
}

// a new ctx over caller memory (no launches): argument checks + workspace carving
static polylla_status new_ctx(const double* xy, int64_t V, const int32_t* tri, int64_t T, int64_t Bmax,
                              bool staging, int64_t R, void* workspace, size_t workspace_bytes_, polylla_ctx** out,
                              bool sorted = false) {
  *out = nullptr;
  if (!xy || !tri || !workspace || V < 3 || T < 1 || Bmax < 0 || Bmax > 3 * T || R < 0)
    return POLYLLA_E_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(xy) & 15) || (reinterpret_cast<uintptr_t>(tri) & 3))
    return POLYLLA_E_INVALID_ARGUMENT;
  if (!index_ok(V, T, Bmax)) return POLYLLA_E_INDEX_OVERFLOW;
  polylla_ctx* p = static_cast<polylla_ctx*>(std::calloc(1, sizeof(polylla_ctx)));
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  Ctx* c = &p->c;
  c->xy = xy;
  c->tri = tri;
  c->V = V;
  c->T = T;
  c->Bmax = Bmax;
  c->staging = staging;
  c->tiling.R = R;  // (carve() derives the tiling: sorted if asked, else grid if R divides T, else contiguous)
  c->tiling.mode = sorted ? kTileSorted : kTileContig;
  if (!carve(c, workspace, workspace_bytes_)) {
    std::free(p);
    return POLYLLA_E_WORKSPACE;
  }
  *out = p;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_build_halfedges_ex(const double* xy, int64_t V, const int32_t* tri, int64_t T,
                                                      int64_t max_border, uint32_t flags, int64_t row_stride,
                                                      void* workspace, size_t workspace_bytes_, polylla_stream stream,
                                                      polylla_ctx** ctx_out) {
  if (!ctx_out) return POLYLLA_E_INVALID_ARGUMENT;
  polylla_ctx* p = nullptr;
  const polylla_status st = new_ctx(xy, V, tri, T, max_border, (flags & POLYLLA_WS_STAGING) != 0, row_stride,
                                    workspace, workspace_bytes_, &p, (flags & POLYLLA_BUILD_SORT) != 0);
  if (st != POLYLLA_OK) return st;
  Ctx* c = &p->c;
  const int n = launch_build(c, S(stream));
  if (n < 0) {
    std::free(p);
    return POLYLLA_E_CUDA;
  }
  c->launches += n;
  c->stage = 1;
  *ctx_out = p;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_build_halfedges(const double* xy, int64_t V, const int32_t* tri, int64_t T,
                                                   void* workspace, size_t workspace_bytes_, polylla_stream stream,
                                                   polylla_ctx** ctx_out) {
  return polylla_build_halfedges_ex(xy, V, tri, T, 3 * T, POLYLLA_WS_STAGING, 0, workspace, workspace_bytes_,
                                    stream, ctx_out);
}

POLYLLA_API polylla_status polylla_check_manifold(polylla_ctx* p, polylla_stream stream) {
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  if (p->c.stage < 1) return POLYLLA_E_CALL_ORDER;
  if (3 * p->c.T + p->c.Bmax > 0x7fffffffLL) return POLYLLA_E_INDEX_OVERFLOW;  // (its slots hold int32 ids + a flag)
  const int n = launch_check_manifold(&p->c, S(stream));
  if (n < 0) return POLYLLA_E_CUDA;
  p->c.launches += n;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_label(polylla_ctx* p, polylla_stream stream) {
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  if (p->c.stage != 1) return POLYLLA_E_CALL_ORDER;
  const int n = launch_label(&p->c, S(stream));
  if (n < 0) return POLYLLA_E_CUDA;
  p->c.launches += n;
  p->c.stage = 2;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_generate(polylla_ctx* p, polylla_stream stream) {
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  if (p->c.stage != 2) return POLYLLA_E_CALL_ORDER;
  const int n = launch_generate(&p->c, S(stream));
  if (n < 0) return POLYLLA_E_CUDA;
  p->c.launches += n;
  p->c.stage = 3;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_label_generate_paper(polylla_ctx* p, polylla_stream stream) {
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  if (p->c.stage != 1) return POLYLLA_E_CALL_ORDER;
  if (3 * p->c.T + p->c.Bmax > 0x7fffffffLL) return POLYLLA_E_INDEX_OVERFLOW;  // (the ablation keeps int32 ids)
  const int n = launch_paper(&p->c, S(stream));
  if (n < 0) return POLYLLA_E_CUDA;
  p->c.launches += n;
  p->c.stage = 3;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_get_counts(polylla_ctx* p, polylla_stream stream, polylla_counts* out) {
  if (!p || !out) return POLYLLA_E_INVALID_ARGUMENT;
  Ctx* c = &p->c;
  if (c->stage < 1) return POLYLLA_E_CALL_ORDER;
  DevCounters h{};
  if (cudaMemcpyAsync(&h, c->ctr, sizeof(h), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
      cudaStreamSynchronize(S(stream)) != cudaSuccess)
    return POLYLLA_E_CUDA;
  polylla_counts r{};
  r.n_vertices = c->V;
  r.n_triangles = c->T;
  r.n_border = h.n_border;
  r.n_halfedges = 3 * c->T + (int64_t)h.n_border;
  r.n_polygons = c->stage >= 3 ? h.P : 0;
  r.n_loop_entries = c->stage >= 3 ? h.L : 0;
  r.n_tips = h.n_tips;
  r.n_flips = h.n_flips;
  r.n_leftover = h.n_left;
  r.n_deferred = h.n_def;
  r.n_seed_deferred = h.n_sdef;
  r.status = (int32_t)map_status(h.status);
  c->host_counts = r;
  if (c->stage == 3) c->stage = 4;
  *out = r;
  return (polylla_status)r.status;
}

POLYLLA_API polylla_status polylla_get_polygons(polylla_ctx* p, uint32_t* offsets, int64_t offsets_cap, int32_t* loops,
                                                int64_t loops_cap, int32_t* origin, uint32_t* twin, uint32_t* next,
                                                uint32_t* prev, polylla_stream stream) {
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  Ctx* c = &p->c;
  if (c->stage < 3) return POLYLLA_E_CALL_ORDER;
  if ((origin || twin || next) && c->stage < 4) return POLYLLA_E_CALL_ORDER;  // H needs get_counts
  if ((offsets != nullptr) != (loops != nullptr)) return POLYLLA_E_INVALID_ARGUMENT;
  // prev is built by a scatter kernel (prev[next[e]] = e): into the caller's array when it
  // is device memory, else into dead workspace scratch (the leftover-key region, 24T bytes
  // >= 4H) and copied out like origin/twin/next -- a kernel must never store to a host
  // pointer
  hid* prev_dev = nullptr;
  if (prev) {
    cudaPointerAttributes pa{};
    const bool on_dev = cudaPointerGetAttributes(&pa, prev) == cudaSuccess &&
                        (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
    cudaGetLastError();  // (clear a failed query of an unregistered host pointer)
    prev_dev = on_dev ? prev : reinterpret_cast<hid*>(c->left_key);
    if (!on_dev && c->stage < 4) return POLYLLA_E_CALL_ORDER;  // the copy-out needs H (get_counts)
  }
  const size_t hb = (size_t)c->host_counts.n_halfedges * 4;
  if (offsets || prev_dev) {
    const int n = launch_extract(c, offsets, offsets ? offsets_cap : -1, loops, loops ? loops_cap : -1, prev_dev,
                                 S(stream));
    if (n < 0) return POLYLLA_E_CUDA;
    c->launches += n;
    if (offsets) c->extracted = true;
  }
  if (prev && prev_dev != prev && cudaMemcpyAsync(prev, prev_dev, hb, cudaMemcpyDefault, S(stream)) != cudaSuccess)
    return POLYLLA_E_CUDA;
  if (origin && cudaMemcpyAsync(origin, c->origin, hb, cudaMemcpyDefault, S(stream)) != cudaSuccess)
    return POLYLLA_E_CUDA;
  if (twin && cudaMemcpyAsync(twin, c->twin, hb, cudaMemcpyDefault, S(stream)) != cudaSuccess)
    return POLYLLA_E_CUDA;
  if (next && cudaMemcpyAsync(next, c->next, hb, cudaMemcpyDefault, S(stream)) != cudaSuccess)
    return POLYLLA_E_CUDA;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_get_triangle_polygons(polylla_ctx* p, int32_t* poly_of_tri, polylla_stream stream) {
  if (!p || !poly_of_tri) return POLYLLA_E_INVALID_ARGUMENT;
  Ctx* c = &p->c;
  if (!c->extracted) return POLYLLA_E_CALL_ORDER;
  const int n = launch_regions(c, poly_of_tri, 0, S(stream));
  if (n < 0) return POLYLLA_E_CUDA;
  c->launches += n;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_get_triangle_regions(polylla_ctx* p, int32_t* region_of_tri, polylla_stream stream) {
  if (!p || !region_of_tri) return POLYLLA_E_INVALID_ARGUMENT;
  Ctx* c = &p->c;
  if (c->stage < 2) return POLYLLA_E_CALL_ORDER;  // F0 is complete after polylla_label
  const int n = launch_regions(c, region_of_tri, 1, S(stream));
  if (n < 0) return POLYLLA_E_CUDA;
  c->launches += n;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_get_views(polylla_ctx* p, polylla_views* v) {
  if (!p || !v) return POLYLLA_E_INVALID_ARGUMENT;
  if (p->c.stage < 1) return POLYLLA_E_CALL_ORDER;
  const Ctx* c = &p->c;
  v->origin = c->origin;
  v->twin = c->twin;
  v->next = c->next;
  v->lcode = c->lcode;
  v->frontier0 = c->F0;
  v->frontier1 = c->F1;
  v->seed_bits = c->S;
  v->seeds = c->seeds;
  v->tips = c->tips;
  return POLYLLA_OK;
}

POLYLLA_API polylla_status polylla_set_debug(polylla_ctx* p, uint32_t* next_pre) {
  if (!p) return POLYLLA_E_INVALID_ARGUMENT;
  p->c.next_pre = next_pre;
  return POLYLLA_OK;
}

// End to end from host buffers, pipelined inside one mesh:
//   up stream   : H2D xy, then tri in kRunChunks chunks of whole build tiles
//   `stream`    : k_tile over each chunk as soon as it has landed, then the rest of the
//                 build, label, generate (one host sync for the counts), extraction
//   down stream : D2H of each chunk's origin rows right behind its k_tile (full duplex:
//                 overlaps the upload of the next chunks), of twin once the build is done
//                 (overlaps label/generate), then the border rows, next and the CSR.
constexpr int kRunChunks = 8;

namespace {
struct RunRes {  // streams and events of one run_host call, released on every exit path
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t ev[2 * kRunChunks + 4] = {};
  int nev = 0;
  bool ok = true;
  cudaEvent_t make() {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) ok = false;
    ev[nev++] = e;
    return e;
  }
  ~RunRes() {
    if (up) cudaStreamSynchronize(up);
    if (down) cudaStreamSynchronize(down);
    for (int i = 0; i < nev; ++i)
      if (ev[i]) cudaEventDestroy(ev[i]);
    if (up) cudaStreamDestroy(up);
    if (down) cudaStreamDestroy(down);
  }
};
}  // namespace

POLYLLA_API polylla_status polylla_run_host(const double* xy_host, int64_t V, const int32_t* tri_host, int64_t T,
                                            void* workspace, size_t workspace_bytes_, uint32_t* offsets_host,
                                            int64_t offsets_cap, int32_t* loops_host, int64_t loops_cap,
                                            int32_t* origin_host, uint32_t* twin_host, uint32_t* next_host,
                                            int64_t halfedge_cap, polylla_counts* counts, polylla_stream stream) {
  if (!xy_host || !tri_host || !workspace || !offsets_host || !loops_host || !counts || V < 3 || T < 1)
    return POLYLLA_E_INVALID_ARGUMENT;
  if (!index_ok(V, T, 3 * T)) return POLYLLA_E_INDEX_OVERFLOW;
  Ctx probe{};
  probe.V = V;
  probe.T = T;
  probe.Bmax = 3 * T;
  probe.staging = true;
  if (!carve(&probe, workspace, workspace_bytes_)) return POLYLLA_E_WORKSPACE;
  polylla_ctx* p = nullptr;
  polylla_status st =
      new_ctx(probe.xy_stage, V, probe.tri_stage, T, 3 * T, true, 0, workspace, workspace_bytes_, &p);
  if (st != POLYLLA_OK) return st;
  Ctx* c = &p->c;
  cudaStream_t s = S(stream);
  polylla_status out = POLYLLA_OK;
  {
    RunRes r;
    if (cudaStreamCreateWithFlags(&r.up, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&r.down, cudaStreamNonBlocking) != cudaSuccess) {
      polylla_destroy(p);
      return POLYLLA_E_CUDA;
    }
    const int64_t tiles = (T + kBuildTileTris - 1) / kBuildTileTris;
    const int nch = (int)(tiles < kRunChunks ? tiles : kRunChunks);
    cudaEvent_t ev_start = r.make(), ev_rest = r.make(), ev_ext = r.make();
    cudaEvent_t ev_up[kRunChunks], ev_tile[kRunChunks];
    for (int i = 0; i < nch; ++i) {
      ev_up[i] = r.make();
      ev_tile[i] = r.make();
    }
    if (!r.ok) {
      polylla_destroy(p);
      return POLYLLA_E_CUDA;
    }
    bool cuda_ok = true;
    auto chk = [&](cudaError_t e) { cuda_ok = cuda_ok && e == cudaSuccess; };
    chk(cudaEventRecord(ev_start, s));  // the side streams start after the caller's prior work
    chk(cudaStreamWaitEvent(r.up, ev_start, 0));
    chk(cudaStreamWaitEvent(r.down, ev_start, 0));
    chk(cudaMemcpyAsync(probe.xy_stage, xy_host, (size_t)V * 16, cudaMemcpyHostToDevice, r.up));
    if (launch_build_begin(c, s) != 0) cuda_ok = false;
    int64_t launches = 0;
    for (int i = 0; i < nch && cuda_ok; ++i) {
      const int64_t t0 = tiles * i / nch, t1 = tiles * (i + 1) / nch;
      const int64_t f0 = t0 * kBuildTileTris, f1 = t1 * kBuildTileTris < T ? t1 * kBuildTileTris : T;
      chk(cudaMemcpyAsync(probe.tri_stage + 3 * f0, tri_host + 3 * f0, (size_t)(f1 - f0) * 12, cudaMemcpyHostToDevice,
                          r.up));
      chk(cudaEventRecord(ev_up[i], r.up));
      chk(cudaStreamWaitEvent(s, ev_up[i], 0));
      const int n = launch_build_tiles(c, s, t0, t1);
      if (n < 0) cuda_ok = false;
      launches += n;
      chk(cudaEventRecord(ev_tile[i], s));
      if (origin_host) {  // interior origin rows of the chunk are final after its k_tile
        chk(cudaStreamWaitEvent(r.down, ev_tile[i], 0));
        chk(cudaMemcpyAsync(origin_host + 3 * f0, c->origin + 3 * f0, (size_t)(f1 - f0) * 12, cudaMemcpyDeviceToHost,
                            r.down));
      }
    }
    if (cuda_ok) {
      const int n = launch_build_rest(c, s);
      if (n < 0) cuda_ok = false;
      launches += n;
      chk(cudaEventRecord(ev_rest, s));
      if (twin_host) {  // interior twins are final after the leftover match and the border ranking
        chk(cudaStreamWaitEvent(r.down, ev_rest, 0));
        chk(cudaMemcpyAsync(twin_host, c->twin, (size_t)(3 * T) * 4, cudaMemcpyDeviceToHost, r.down));
      }
    }
    if (!cuda_ok) {
      polylla_destroy(p);
      return POLYLLA_E_CUDA;
    }
    c->launches += launches;
    c->stage = 1;
    if ((st = polylla_label(p, stream)) != POLYLLA_OK || (st = polylla_generate(p, stream)) != POLYLLA_OK) {
      polylla_destroy(p);
      return st;
    }
    st = polylla_get_counts(p, stream, counts);  // the one host sync (the side streams keep copying)
    if (st != POLYLLA_OK) {
      polylla_destroy(p);
      return st;
    }
    const int64_t P = counts->n_polygons, L = counts->n_loop_entries, H = counts->n_halfedges;
    if (offsets_cap < P + 1 || loops_cap < L || ((origin_host || twin_host || next_host) && halfedge_cap < H)) {
      polylla_destroy(p);
      return POLYLLA_E_CAPACITY;
    }
    // extraction into the workspace staging, then exact-size copies
    if (launch_extract(c, nullptr, T + 1, c->loops, 3 * T, nullptr, s) < 0) out = POLYLLA_E_CUDA;
    chk(cudaEventRecord(ev_ext, s));
    chk(cudaStreamWaitEvent(r.down, ev_ext, 0));  // (after generate too: next is final)
    const size_t hb = (size_t)(H - 3 * T) * 4;     // border rows
    if (origin_host && hb) chk(cudaMemcpyAsync(origin_host + 3 * T, c->origin + 3 * T, hb, cudaMemcpyDeviceToHost, r.down));
    if (twin_host && hb) chk(cudaMemcpyAsync(twin_host + 3 * T, c->twin + 3 * T, hb, cudaMemcpyDeviceToHost, r.down));
    if (next_host) chk(cudaMemcpyAsync(next_host, c->next, (size_t)H * 4, cudaMemcpyDeviceToHost, r.down));
    chk(cudaMemcpyAsync(offsets_host, c->offsets, (size_t)(P + 1) * 4, cudaMemcpyDeviceToHost, r.down));
    chk(cudaMemcpyAsync(loops_host, c->loops, (size_t)L * 4, cudaMemcpyDeviceToHost, r.down));
    chk(cudaStreamSynchronize(r.down));
    chk(cudaStreamSynchronize(r.up));
    if (!cuda_ok) out = POLYLLA_E_CUDA;
    // (RunRes releases the streams and events)
  }
  polylla_destroy(p);
  return out;
}

POLYLLA_API void polylla_destroy(polylla_ctx* p) { std::free(p); }

POLYLLA_API void polylla_profile_enable(int on) {
  g_prof = on != 0;
  g_entries.clear();
  g_pool_used = 0;
  g_open = nullptr;
}

POLYLLA_API int polylla_profile_read(const char** names, double* total_ms, int64_t* count, int cap) {
  std::map<std::string, std::pair<double, int64_t>> acc;
  std::vector<std::string> order;
  for (const ProfEntry& e : g_entries) {
    if (cudaEventSynchronize(e.b) != cudaSuccess) return -1;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    auto it = acc.find(e.name);
    if (it == acc.end()) {
      order.push_back(e.name);
      acc[e.name] = {ms, 1};
    } else {
      it->second.first += ms;
      it->second.second += 1;
    }
  }
  int n = 0;
  static std::vector<std::string> keep;  // stable storage for the returned names
  keep = order;
  for (const std::string& k : keep) {
    if (n >= cap) break;
    names[n] = k.c_str();
    total_ms[n] = acc[k].first;
    count[n] = acc[k].second;
    ++n;
  }
  g_entries.clear();
  g_pool_used = 0;
  g_open = nullptr;
  return n;
}

POLYLLA_API int64_t polylla_launch_count(const polylla_ctx* p) { return p ? p->c.launches : 0; }

POLYLLA_API const char* polylla_status_string(polylla_status s) {
  switch (s) {
    case POLYLLA_OK: return "ok";
    case POLYLLA_E_INVALID_ARGUMENT: return "invalid argument";
    case POLYLLA_E_DANGLING_INDEX: return "dangling vertex index";
    case POLYLLA_E_DEGENERATE_TRI: return "degenerate triangle";
    case POLYLLA_E_NON_MANIFOLD_EDGE: return "non-manifold edge";
    case POLYLLA_E_NON_MANIFOLD_VERTEX: return "non-manifold boundary vertex";
    case POLYLLA_E_INDEX_OVERFLOW: return "half-edge index overflow";
    case POLYLLA_E_WORKSPACE: return "workspace too small or misaligned";
    case POLYLLA_E_WALK_BOUND: return "walk bound exceeded";
    case POLYLLA_E_UNSEEDED_LOOP: return "frontier loop without a seed";
    case POLYLLA_E_CALL_ORDER: return "call order";
    case POLYLLA_E_CUDA: return "CUDA error";
    case POLYLLA_E_CAPACITY: return "output capacity too small";
  }
  return "unknown";
}

}  // extern "C"
