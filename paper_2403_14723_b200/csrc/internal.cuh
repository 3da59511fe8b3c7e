// internal.cuh -- shared declarations of the libpolylla.so kernels (CUDA, sm_100a).
//
// Data layout in HBM (all inside the caller's workspace, see carve() in capi.cu):
//   origin/twin/next : int32 SoA [H_max], H_max = 6T (worst case B = 3T)
//   lcode            : uint8 [T]   k* of each triangle (longest half-edge 3f+k*)
//   F0, F1, S, C     : uint32 bit-vectors over the interior half-edges [0, 3T)
//                      (frontier before/after repair, seed, canonical seed)
//   len              : int32 [3T]  loop length, written only at canonical seeds
//   TB, SDB          : uint32 bit-vectors: barrier tips, seeds for the global seed walk
//   leftover keys/ids (per-tile segments), global edge hash, border-vertex map vmap[V], tips, mids, scan sums,
//   seeds/offsets/loops staging, input staging (run_host).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "polylla.h"

namespace polylla {

// Half-edge ids are UNSIGNED 32-bit (capacity beyond int32):
// H = 3T + B <= 2^32 - 2, so 0xFFFFFFFF stays free as the "none" sentinel.  Vertex ids
// (origin, loops, the input triangles) and triangle ids stay int32 (V, T < 2^31).
using hid = uint32_t;
constexpr hid kNoHe = 0xFFFFFFFFu;
constexpr int64_t kMaxHalfedges = 0xFFFFFFFELL;  // 3T + B must not exceed this

// ------------------------------------------------------------------ status bits
enum : uint32_t {
  ST_DANGLING = 1u << 0,
  ST_DEGENERATE = 1u << 1,
  ST_NONMANIFOLD_EDGE = 1u << 2,
  ST_NONMANIFOLD_VERTEX = 1u << 3,
  ST_WALK = 1u << 4,
  ST_UNSEEDED = 1u << 5,
  ST_CAPACITY = 1u << 6,
  ST_OVERFLOW = 1u << 7,
  ST_INTERNAL = 1u << 8,
  ST_BORDER_CAP = 1u << 9,  // B exceeds the workspace's border bound (polylla_workspace_bytes_ex)
};

// device-side counters (zeroed at the start of every build)
struct DevCounters {
  uint32_t status;
  uint32_t n_left;   // leftover half-edges (twin not in the build tile)
  uint32_t n_border; // B
  int32_t n_tips;
  int32_t n_flips;
  int32_t P;         // polygons (<= T < 2^31)
  uint32_t L;        // loop entries (<= 3T)
  uint32_t n_f1;     // #interior F1 half-edges
  uint32_t hash_cap; // capacity (pow2 <= 2^31) of the leftover hash for this run
  uint32_t n_def;    // half-edges deferred by k_tile to the label fixup
  uint32_t n_sdef;   // seeds walked by k_seed_walk (deferred + repair halves)
  uint32_t n_cross;  // (regions, grid tiling) pairs crossing the union-find tiles
  unsigned long long hash_scale;  // leftover-hash home slot = (lo * hash_scale) >> 32 (cap / V in 32.32 fixed point)
  int32_t pad[2];
};

// The build tiling (k_tile's tiles and the per-tile list segments).  Contiguous (R = 0):
// tile t = triangles [2048 t, 2048 t + 2048).  Grid (row-major input whose triangle rows
// are R triangles long, e.g. R = 2(s-1) for the Alg. 13 grids of PAPER.md L910-941):
// tile (tr, tc) = triangle rows [16 tr, +16) x columns [128 tc, +128), numbered
// t = tr * ntc + tc; its local triangle u = 128 r + c is triangle (16 tr + r) R + 128 tc + c.
// A thin strip of one row cuts a third of all edges; a 16 x 128 patch cuts ~3%.
constexpr int kGridTW = 128, kGridTH = 16, kGridTWShift = 7;  // kGridTW * kGridTH = 2048 triangles
// Sorted tiling (POLYLLA_BUILD_SORT, any input order): the build first orders the
// triangles by the Morton cell of their centroid (a counting sort into ~T/16 cells of the
// bounding box) and tile t takes triangles perm[2048 t .. 2048 t + 2048).
enum : int { kTileContig = 0, kTileGrid = 1, kTileSorted = 2 };
struct Tiling {
  int mode = kTileContig;
  int64_t R = 0;      // (grid) triangles per row
  int64_t nrows = 0;  // (grid) T / R
  int64_t ntc = 0;    // (grid) column tiles per band: ceil(R / 128)
  int64_t ntiles = 0;
  const int32_t* perm = nullptr;  // (sorted) triangle order
};
struct TileGeom {
  int64_t base;       // global triangle of local triangle 0
  int64_t seg;        // first entry of the tile's list segment (3 x its triangles, contiguous over tiles)
  int32_t nrows, ncols;  // grid tiles: rows / columns present
};
__host__ __device__ __forceinline__ TileGeom contig_geom(int64_t T, int64_t tile) {
  TileGeom r;
  r.base = tile * 2048;
  r.seg = 3 * r.base;
  const int64_t n = T - r.base < 2048 ? T - r.base : 2048;
  r.nrows = (int32_t)n;  // (contiguous: nrows = triangles present, ncols unused)
  r.ncols = 0;
  return r;
}
__host__ __device__ __forceinline__ TileGeom tile_geom(const Tiling& g, int64_t T, int64_t tile) {
  if (g.mode != kTileGrid) return contig_geom(T, tile);  // (sorted tiles: positions in perm)
  TileGeom r;
  const int64_t tr = tile / g.ntc, tc = tile - tr * g.ntc;
  const int64_t row0 = tr * kGridTH, col0 = tc * kGridTW;
  r.nrows = (int32_t)(g.nrows - row0 < kGridTH ? g.nrows - row0 : kGridTH);
  r.ncols = (int32_t)(g.R - col0 < kGridTW ? g.R - col0 : kGridTW);
  r.base = row0 * g.R + col0;
  r.seg = 3 * (row0 * g.R + col0 * r.nrows);
  return r;
}
Tiling make_tiling(int64_t T, int64_t R, bool sorted);  // sorted > grid (R > 0 dividing T) > contiguous

struct Ctx {
  // inputs
  const double* xy;
  const int32_t* tri;
  int64_t V, T;
  int64_t Hmax;  // 3T + the border bound (6T by default)
  int64_t Bmax;  // border bound of the workspace layout
  bool staging;  // the layout holds run_host's staging regions
  Tiling tiling; // the build tiling (contiguous unless a row stride was given)
  uint32_t* BB;  // [n_words] unmatched leftovers (grid/sorted tiling: the border ranking by bit scan)
  uint32_t* sort_key;   // (sorted tiling) [T] Morton cell of each triangle
  uint32_t* sort_hist;  // (sorted tiling) [kSortCells] cell counts, then cursors
  unsigned long long* sort_bbox;  // (sorted tiling) [4] order-preserving encodings of min/max x, y
  // workspace views
  int32_t* origin;   // vertex ids
  hid *twin, *next;
  uint8_t* lcode;
  uint32_t *F0, *F1, *S, *C;
  uint8_t* len;     // [3T] loop length at canonical seeds, min(n, kLenEsc) (bytes: its sparse reads and
                    // writes touch a quarter of the sectors of an int32 array)
  int32_t* wlen;    // [n_words] sum of loop lengths of the canonical seeds of each C word
  unsigned long long* left_key;
  hid* left_e;
  hid* def_e;       // [3T] half-edges deferred by k_tile (per-tile segments at 3 * tile * 2048)
  uint32_t* SDB;    // [n_words] seeds for the global seed walk (deferred by k_tile / the fixup, repair halves)
  uint32_t* TB;     // [n_words] barrier tips (incoming frontier half-edge e, next[e] == twin[e])
  int32_t* cnt_ld;  // [2 * tiles] per-tile leftover / deferred counts
  int32_t* tsum;    // [3 * tiles] per-tile #canonical seeds, sum of loop lengths, #F1
  uint32_t* tbase;  // [2 * tiles] per-tile exclusive prefix of polygons / loop entries
  uint32_t* bcnt;   // [tiles] per-tile border half-edge count, then (in place) its base
  void* ehash;      // leftover-edge hash slots [hash_cap_max], u32 (3T < 2^31) or u64 (capacity chosen on device)
  hid* vmap;        // [V] border half-edge leaving each border vertex (written at border vertices only)
  int64_t hash_cap_max;
  hid* tips;        // [V]
  hid* aff;         // [2V] affected (outgoing half-edge) per tip side
  hid* mids;        // [2V]
  long long* scan_a;  // per-block sums (count)
  long long* scan_b;  // per-block sums (aux)
  long long* scan_c;  // per-block sums (F1 popcount)
  hid* seeds;         // [T]
  uint32_t* offsets;  // [T+1]
  int32_t* loops;     // [3T]  (run_host staging)
  double* xy_stage;   // [2V]  (run_host staging)
  int32_t* tri_stage; // [3T]
  DevCounters* ctr;
  hid* next_pre;      // optional debug copy
  // host state
  int stage;          // 1 built, 2 labelled, 3 generated, 4 counted
  bool extracted;     // polylla_get_polygons wrote the polygon seeds
  int64_t launches;
  polylla_counts host_counts;
  int64_t n_words;    // ceil(3T/32)
  int64_t scan_blocks;
};

// optional per-kernel timing (polylla_profile_*): events recorded around launches
void prof_mark(cudaStream_t s, const char* name);  // start of kernel `name` (ends at the next mark)
void prof_end(cudaStream_t s);

// workspace
constexpr int64_t kSortCells = int64_t(1) << 16;  // Morton cells (8 bits per axis) for the sorted tiling
size_t workspace_bytes(int64_t V, int64_t T, int64_t Bmax, bool staging, int64_t R = 0, bool sorted = false);
bool carve(Ctx* c, void* ws, size_t bytes);  // layout from c->V, c->T, c->Bmax, c->staging

// launchers (each returns the number of kernel launches issued, < 0 on CUDA error)
int launch_build(Ctx* c, cudaStream_t s);  // = begin + tiles [0, ntiles) + rest
int launch_build_begin(Ctx* c, cudaStream_t s);
int launch_build_tiles(Ctx* c, cudaStream_t s, int64_t t0, int64_t t1);
int launch_build_rest(Ctx* c, cudaStream_t s);
int launch_label(Ctx* c, cudaStream_t s);
int launch_generate(Ctx* c, cudaStream_t s);
int launch_extract(Ctx* c, uint32_t* offsets, int64_t offsets_cap, int32_t* loops, int64_t loops_cap,
                   hid* prev, cudaStream_t s);
int launch_regions(Ctx* c, int32_t* out, int mode, cudaStream_t s);  // mode 0: polygon ids, 1: F0 regions
int launch_check_manifold(Ctx* c, cudaStream_t s);
int launch_paper(Ctx* c, cudaStream_t s);  // the paper's LLK..OSK + Scan sequence (NEXT-2 ablation)

// Programmatic dependent launch (PDL): the hot-path kernels are launched with
// programmatic stream serialisation, so a kernel's CTAs are scheduled while its
// predecessor's last wave still runs; each kernel waits (griddepcontrol.wait: the
// predecessor grid complete and its writes visible) before touching any memory, then
// lets its own successor launch.  POLYLLA_PDL=0 builds plain launches (A/B).
#ifndef POLYLLA_PDL
#define POLYLLA_PDL 1
#endif
__device__ __forceinline__ void pdl_enter() {
#if POLYLLA_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KP, typename... A>
inline void launch_k(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A... a) {
#if POLYLLA_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KP>(a)...);  // (errors: cudaGetLastError at the launcher's end)
#else
  k<<<grid, block, smem, s>>>(static_cast<KP>(a)...);
#endif
}

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ hid next_in(hid e) {  // 3f + (k+1)%3
  const hid k = e % 3u;
  return k == 2 ? e - 2 : e + 1;
}
__device__ __forceinline__ hid prev_in(hid e) {  // 3f + (k+2)%3
  const hid k = e % 3u;
  return k == 0 ? e + 2 : e - 1;
}
__device__ __forceinline__ bool bit_of(const uint32_t* w, hid e) { return (w[e >> 5] >> (e & 31)) & 1u; }

__device__ __forceinline__ void raise_status(DevCounters* c, uint32_t bits) { atomicOr(&c->status, bits); }

__device__ __forceinline__ uint32_t mix32(uint32_t a, uint32_t b) {
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u + (a << 6) + (a >> 2));
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

constexpr uint32_t kEmpty = 0xFFFFFFFFu;   // empty hash slot
constexpr uint32_t kLenEsc = 255;          // len[]: a loop of >= 255 entries (its length is counted by walking it)
__device__ __forceinline__ uint8_t len_code(int64_t n) { return (uint8_t)(n < (int64_t)kLenEsc ? n : kLenEsc); }
constexpr int kBuildTileTris = 2048;     // triangles per k_tile tile (list segments are 3 * 2048 wide)

// Block -> tile schedule of the per-tile kernels.  POLYLLA_REVERSE_TILES (a test variant,
// tests/variants.py) runs the tiles in reverse order: results must not depend on it.
__device__ __forceinline__ int64_t sched_tile(int64_t i, int64_t ntiles) {
#ifdef POLYLLA_REVERSE_TILES
  return ntiles - 1 - i;
#else
  (void)ntiles;
  return i;
#endif
}

// Set bits of a bit-vector, spread over warps: warp g of the grid scans kBitChunk-word
// chunks g, g + G, ... and expands the set bits into its shared queue q (kBitQueue
// entries); each full (or final) queue is handed to f(e, valid) in warp-uniform rounds of
// 32 (all lanes present, so f may use warp collectives; valid is false on the padding
// lanes of the last round; e is then kNoHe).  Returns the number of set bits this warp saw.
#ifndef POLYLLA_BIT_QUEUE
#define POLYLLA_BIT_QUEUE 256  // (64 / 128 / 256 / 512 measured: 256 best for k_seed_walk on config 3)
#endif
constexpr int kBitQueue = POLYLLA_BIT_QUEUE;  // small: the walks that follow live on L1 hits (shared memory shrinks L1)
#ifndef POLYLLA_BIT_CHUNK
#define POLYLLA_BIT_CHUNK 32
#endif
constexpr int kBitChunk = POLYLLA_BIT_CHUNK;  // words per warp chunk (<= 32; 8 and 4 measured slower)
static_assert(kBitChunk >= 1 && kBitChunk <= 32, "one word per lane");
// (WHOLE: each full or final queue is handed to f(q, fill) at once, all lanes present)
template <bool WHOLE = false, class F>
__device__ __forceinline__ int warp_foreach_bit(const uint32_t* __restrict__ bv, int64_t n_words, hid* q, F f) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int fill = 0, seen = 0;
  auto flush = [&]() {
    __syncwarp();
    if constexpr (WHOLE) {
      f(q, fill);
    } else {
      for (int base = 0; base < fill; base += 32) f(base + lane < fill ? q[base + lane] : kNoHe, base + lane < fill);
    }
    __syncwarp();
    fill = 0;
  };
  // interleaved kBitChunk-word chunks: at any time the grid works inside one window of
  // the mesh (nwarps * kBitChunk * 32 half-edges), which keeps the walks' next/twin
  // lines in L2
  for (int64_t w0 = gwarp * kBitChunk; w0 < n_words; w0 += nwarps * kBitChunk) {
    const int64_t w = w0 + lane;
    uint32_t bits = (lane < kBitChunk && w < n_words) ? bv[w] : 0u;
    while (__any_sync(0xffffffffu, bits != 0u)) {
      const int c = __popc(bits);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += a;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (fill + tot > kBitQueue && fill > 0) flush();
      // append as many bits as fit (a dense group may need several passes)
      const int room = kBitQueue - fill, excl = incl - c;
      int take = room - excl;
      take = take < 0 ? 0 : (take > c ? c : take);
      for (int p = fill + excl, k = 0; k < take; ++k, bits &= bits - 1) q[p++] = (hid)(w * 32 + __ffs(bits) - 1);
      const int added = tot < room ? tot : room;
      fill += added;
      seen += added;
      if (fill == kBitQueue) flush();
    }
  }
  if (fill) flush();
  return seen;
}

}  // namespace polylla
