// build.cu -- half-edge construction on the device,
// fused with the longest-edge labelling (Alg. 2 / Alg. 7).
//
// The paper builds the half-edge structure on the CPU and copies it over (L273).  Here
// one pass over triangle tiles does everything that only needs the tile:
//
//   k_tile  (one CTA per tile of kTileTris triangles, input read once, coalesced)
//     - orientation fix (signed area in FP64, no FMA), dangling/degenerate checks;
//     - Lcode[f] = first argmax_k |e_k|^2 over the half-edges 3f+k (tie -> lower id, R7);
//     - origin[3f+k] = tri'[f][k] (the oriented tile, written back coalesced);
//     - twin matching inside the tile through a shared-memory hash on the undirected
//       key (min, max) -- Morton-ordered meshes keep ~96% of twins inside a tile;
//     - frontier/seed classification and the unlink rewire of every half-edge whose
//       rotation walk stays inside the tile (label.cu completes the others);
//     - polygons that close inside the tile: canonical seed and loop length;
//     - half-edges whose twin is outside the tile go to the tile's leftover segment,
//       those whose rotation leaves it to its deferred segment.
//   k_left_insert                      -- global hash over the leftovers only;
//   k_border_rank / _scan / _emit      -- border ids 3T + rank(e) (R9), twin/origin of
//                                         border half-edges, border-vertex map;
//   k_border_next                      -- next(b) = border half-edge leaving target(b).
#include <cstdlib>
#include <mutex>

#include "internal.cuh"

namespace polylla {

constexpr int kTileTris = kBuildTileTris;
constexpr int kTileHE = 3 * kTileTris;   // 6144 half-edges = 192 bit-vector words (e order)
constexpr int kTileQ = 4 * kTileTris;    // quad slots q = 4t + k (slot 3: copy of vertex 0 / unused)
#ifndef POLYLLA_TILE_SLOTS
#define POLYLLA_TILE_SLOTS 24000  // (a multiple of 8, >= 4,096; measured 12,288 / 15,360 / 19,456 / 21,504 / 22,528 / 24,000)
#endif
// hash slots of 16 bits (only the lo->hi halves insert: 3,072 keys, load 0.13); the table
// overlays the P3-P6 arrays.  The tile's shared memory also decides the L1 left for the
// coordinate gathers (the carveout is the smallest that holds two CTAs): 105 KB per CTA
// (228 KB carveout, 28 KB of L1) -> 90 KB (196 KB, 60 KB of L1) cut k_tile by 11% on
// config 3; within the 196 KB carveout a larger table then pays (fewer collision losers
// and probing lookups): 99,200 B per CTA with 24,000 slots, the most that stays inside it.
constexpr int kTileSlots = POLYLLA_TILE_SLOTS;
static_assert(kTileSlots % 8 == 0 && kTileSlots >= 2 * kBuildTileTris, "slot count: uint4 clears, load < 1/2");
#ifndef POLYLLA_TILE_THREADS
#define POLYLLA_TILE_THREADS 768
#endif
constexpr int kTileThreads = POLYLLA_TILE_THREADS;
constexpr int kTileWords = kTileHE / 32; // 192
constexpr int kTriIters = (kTileTris + kTileThreads - 1) / kTileThreads;  // 768: 3 (the third: threads < 512)
static_assert(kTileThreads % 32 == 0 && (kTileTris - (kTriIters - 1) * kTileThreads) % 32 == 0,
              "warp-uniform last triangle iteration");
static_assert(4 * kTriIters <= 32, "per-lane pending bit masks");
constexpr int kHeIters = (kTileHE + kTileThreads - 1) / kTileThreads;     // 768: 8 exactly
constexpr bool kHePartial = kTileHE % kTileThreads != 0;                  // (other thread counts)
static_assert(kTileThreads % 3 != 2 && (kTileHE % kTileThreads) % 32 == 0, "half-edge loops: q_step below");
// quad of half-edge j + kTileThreads from the quad q of j (no division): 768 = 3 * 256
// -> q + 1024; 1024 = 3 * 341 + 1 -> q + 1365, skipping the padding slot k = 3
constexpr int kQStep = 4 * (kTileThreads / 3) + kTileThreads % 3;
__device__ __forceinline__ int q_step(int q) {
  q += kQStep;
  if (kTileThreads % 3 == 1 && (q & 3) == 3) ++q;
  return q;
}
// shared memory (bytes):
//   tri_q int32[kTileQ]   32768  quad layout (v0, v1, v2, v0): half-edge q runs tri_q[q] -> tri_q[q+1]
//   tw_s  int16[kTileQ]   16384  twin as a quad index, -1 = outside the tile (P2-P4b); then, written
//                                over it quad by quad in P4b, nx_q: the local next (quad index),
//                                -1 not walkable, kNxTip | twin for a barrier tip (P4b-P6)
//   lc_s  u8[kTileTris]    2048
//   then one region that changes role after P2c:
//     P0-P2c: slot u16[kTileSlots]       quad index of a lo->hi half-edge, 0xFFFF empty
//     P3-P6 : succ u16[kTileQ] 16384 (pointer jumping in place) |
//             Sw, Cw, Wl, Lm, Dm, SDm, Fw, Tw u32[192] 6144   (Fw, Tw: the frontier / tip
//             words of a grid tile, flushed at the end)
constexpr size_t kOffTw = kTileQ * 4, kOffLc = kOffTw + kTileQ * 2, kOffSlot = kOffLc + kTileTris,
                 kOffWords = kOffSlot + kTileQ * 2,                            // (succ: the first 16 KB of the region)
                 kWordBytes = 8 * (kTileHE / 8),                               // 6,144 B
                 kSeedListBytes = 16 + 2 * (kTileHE / 2),                     // (P6 list: count + u16 seeds)
                 kP3Bytes = kTileQ * 2 + kWordBytes + kSeedListBytes,
                 kRegion = kP3Bytes > kTileSlots * 2 ? kP3Bytes : kTileSlots * 2,
                 kTileSmemGrid = kOffSlot + kRegion,                           // 99,200 B -> 2 CTAs/SM in 196 KB
                 kTileSmem = kTileSmemGrid;
constexpr int kNxTip = 0x4000;  // nx_q: barrier tip (quad indices are < 0x2000)
static_assert(2 * (kTileSmemGrid + 1024) <= 228 * 1024, "two tiles per SM");
static_assert(POLYLLA_TILE_SLOTS != 24000 || 2 * (kTileSmemGrid + 1024) <= 196 * 1024, "the 196 KB carveout");
static_assert(kOffSlot % 16 == 0, "uint4 clears of the slot table");
constexpr unsigned long long kLeftDown = 1ull << 63;    // leftover key: set if origin > target
constexpr unsigned long long kLeftPaired = 1ull << 31;  // leftover key: set once the key's slot holder is paired
constexpr uint32_t kEmpty16 = 0xFFFFu;             // empty 16-bit slot (quad indices are < 8192)
// rotation successors (P3/P4): quad index in the low 13 bits, terminal flags above
constexpr uint16_t kSuccIdx = 0x1FFF, kSuccFront = 0x4000, kSuccUnknown = 0x8000;
#ifndef POLYLLA_TILE_JUMPS
#define POLYLLA_TILE_JUMPS 1  // measured 0 / 2 / 4 (round 2), 1 / 2 / 3 with the in-place jumping: 1 best
#endif
// pointer-jumping rounds (in place: after r rounds a successor is >= 2^r steps ahead); each
// use of a successor then follows up to kTileHops more jumped pointers, so chains up to 16
// steps resolve in-tile
constexpr int kTileJumps = POLYLLA_TILE_JUMPS;
constexpr int kTileHops = (16 >> kTileJumps) - 1;
#ifndef POLYLLA_P6_MAXLEN
#define POLYLLA_P6_MAXLEN 1024  // (a test variant sets it tiny to force the global seed walk)
#endif
constexpr int kP6MaxLen = POLYLLA_P6_MAXLEN;
#ifndef POLYLLA_P6_LIST
#define POLYLLA_P6_LIST 1  // P6 takes the tile's seeds from a list, one per thread (0: kSeedLanes per word)
#endif  // in-tile loop walks longer than this go to k_seed_walk

#ifdef POLYLLA_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
// (__syncthreads_count's result is consumed before the clock is read: clock64() right
// after a plain __syncthreads records the deferred barrier's issue time, not its release)
#define PHASE_MARK(i)                                                       \
  do {                                                                      \
    const int c_ = __syncthreads_count(1); /* result depends on release */  \
    if (threadIdx.x == 0 && c_ > 0) {                                       \
      const long long now_ = clock64();                                     \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(now_ - t_phase_)); \
      t_phase_ = now_;                                                      \
    }                                                                       \
  } while (0)
#else
#define PHASE_MARK(i) do { } while (0)
#endif

// quad encoding of a local half-edge: q = 4*(j/3) + j%3 (bit ops in the walks)
__device__ __forceinline__ int32_t q_of(int32_t j) { const int32_t t = j / 3; return 4 * t + (j - 3 * t); }
__device__ __forceinline__ int32_t j_of(int32_t q) { return 3 * (q >> 2) + (q & 3); }
__device__ __forceinline__ int32_t next_q(int32_t q) { return (q & 3) == 2 ? q - 2 : q + 1; }

// Relaxed CTA-scope atomic load/store on shared memory (plain LDS/STS in SASS): the hash
// slot claim is last-writer-wins by design and is read while collision losers CAS, so
// these accesses are atomics in the memory model rather than data races.
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.cta.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v));
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}

__device__ __forceinline__ void st_relaxed16(uint16_t* p, uint32_t v) {
  asm volatile("st.relaxed.cta.shared.u16 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "h"((uint16_t)v));
}
__device__ __forceinline__ uint32_t ld_relaxed16(const uint16_t* p) {
  uint16_t v;
  asm volatile("ld.relaxed.cta.shared.u16 %0, [%1];" : "=h"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}

__device__ __forceinline__ double sq_len(double2 p, double2 q) {
  // |q - p|^2 = dx*dx + dy*dy, dx = x[target] - x[origin]; IEEE RN, no FMA (R11)
  const double dx = __dsub_rn(q.x, p.x), dy = __dsub_rn(q.y, p.y);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// L2 policy for the randomly gathered coordinates (vertex ids are spatially random)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_xy(const double2* ptr, uint64_t pol) {
  double2 r;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(ptr), "l"(pol));
  return r;
}

// Tile hash on the undirected key (lo, hi): linear probing over 16-bit slots holding the
// quad index of the lo->hi half-edge (origin < target); the hi->lo halves look it up
// read-only.  A slot is verified against the key through tri_q (the slot carries no
// fingerprint: 16-bit slots double the slot count in the same 32 KB, halving the
// collision losers of the claim pass).  The high bits of the product are well mixed.
__device__ __forceinline__ uint32_t tile_hash(uint32_t lo, uint32_t hi) {
  return ((lo * 0x9E3779B1u) ^ hi) * 0x85EBCA6Bu;
}
// home slot: the high bits of hash * kTileSlots (a power of two: the top bits of the hash)
__device__ __forceinline__ uint32_t tile_pos(uint32_t lo, uint32_t hi) { return __umulhi(tile_hash(lo, hi), (uint32_t)kTileSlots); }
__device__ __forceinline__ uint32_t slot_succ(uint32_t p) { return p + 1 == (uint32_t)kTileSlots ? 0u : p + 1; }

// collision loser of the claim pass: CAS (on the 32-bit word holding the 16-bit slot) +
// linear probing from its home slot
#ifdef POLYLLA_PROBE_NOINLINE  // (inlined: k_tile -1% with the 24,000-slot table)
#define POLYLLA_PROBE_ATTR __noinline__
#else
#define POLYLLA_PROBE_ATTR __forceinline__
#endif
__device__ POLYLLA_PROBE_ATTR uint32_t tile_insert_probe(uint16_t* slot, const int32_t* tri_q, int32_t q, uint32_t lo,
                                                   uint32_t hi) {
  uint32_t p = tile_pos(lo, hi);
  for (int probe = 0; probe < kTileSlots; ++probe, p = slot_succ(p)) {
    uint32_t* wp = reinterpret_cast<uint32_t*>(slot + (p & ~1u));
    const int sh = (int)(p & 1) * 16;
    uint32_t word = ld_relaxed(wp);
    uint32_t v = (word >> sh) & 0xFFFFu;
    while (v == kEmpty16) {
      const uint32_t old = atomicCAS(wp, word, (word & ~(0xFFFFu << sh)) | ((uint32_t)q << sh));
      if (old == word) return 0;
      word = old;  // (the other half changed, or this one was taken)
      v = (word >> sh) & 0xFFFFu;
    }
    if ((uint32_t)tri_q[v] == lo && (uint32_t)tri_q[v + 1] == hi) return ST_NONMANIFOLD_EDGE;  // same directed edge twice
  }
  return ST_INTERNAL;
}

// the quad holding key lo -> hi, probing from the slot after its home (the home missed), or -1
__device__ POLYLLA_PROBE_ATTR int32_t tile_lookup_probe(const uint16_t* slot, const int32_t* tri_q, uint32_t lo, uint32_t hi) {
  uint32_t p = tile_pos(lo, hi);
  for (int probe = 1; probe < kTileSlots; ++probe) {
    p = slot_succ(p);
    const uint32_t w = slot[p];
    if (w == kEmpty16) return -1;
    if ((uint32_t)tri_q[w] == lo && (uint32_t)tri_q[w + 1] == hi) return (int32_t)w;
  }
  return -1;
}

// is triangle slot i (t = tid + 768 i) of this thread inside the tile?  For a full tile
// this is compile-time true for all but the last iteration and warp-uniform for the last
// (768 threads: i < 2 always, i = 2 for threads < 512).
template <bool FULL>
__device__ __forceinline__ bool tri_ok(int i, int t, int nt) {
  return FULL ? (i < kTriIters - 1 || threadIdx.x < kTileTris - (kTriIters - 1) * kTileThreads) : t < nt;
}
// local triangle t of a partial tile: contiguous tiles hold a prefix (t < nt); grid tiles a
// nrows x ncols corner of the 16 x 128 patch (t = 128 r + c)
template <bool FULL, bool GRID>
__device__ __forceinline__ bool tri_here(int i, int t, int nt, int nrows, int ncols) {
  if (FULL) return tri_ok<true>(i, t, nt);
  if (GRID) return (i < kTriIters - 1 || threadIdx.x < kTileTris - (kTriIters - 1) * kTileThreads) &&
                   (t & (kGridTW - 1)) < ncols && (t >> kGridTWShift) < nrows;
  return t < nt;
}

// One CTA per tile of kTileTris triangles.  Phases (PAPER.md section in brackets):
//  P0 clear the hash; bulk L2 prefetch of the tile that starts when this one ends
//  P1 per triangle: checks, CCW orientation (R10), longest edge Lcode (Alg. 2/7); the
//     oriented triangle goes to shared memory in quad layout
//  P2 tile-local twin matching in a shared-memory hash on (min, max): the lo->hi halves
//     insert (plain-store claim of the home slot, CAS only for collision losers -- shared
//     atomics cost ~2 cycles per lane), the hi->lo halves look up read-only; the home
//     slot of every half-edge is probed without divergence, only misses loop   [Sec. 4]
//  P3 origin/twin written back coalesced; rotation successor of every half-edge: itself if it
//     is a frontier edge (Alg. 8), else next_in(twin) (sweep_out, R1); a third copy of
//     an edge breaks the twin involution
//  P4 the unlink rewire (Alg. 11) by pointer jumping on the successors (kTileJumps
//     rounds in place, then up to kTileHops jumped hops at each use: chains <= 16 steps); frontier / seed bits (Alg. 8-9); tips (next == twin);
//     half-edges needing a twin outside the tile (or a longer rotation) are deferred
//     to k_label_fixup (label phase)
//  P5 the leftover and deferred lists as per-tile segments (each word ranked by its warp)
//  P6 seeds whose polygon closes inside the tile: landing + loop walk in shared memory
//     -> canonical seed bits and loop lengths (others go to the global seed walk via the
//     bit-vector SDB; tips go to the bit-vector TB)
// Loops are indexed so that no lane divides: triangle t = tid + 768 i, half-edge
// j = tid + 768 i with quad q = q_of(tid) + 1024 i (768 = 3 * 256).
template <bool FULL, int MODE>
__device__ __forceinline__ void tile_body(
    unsigned char* smem_tile, const Tiling tl, const double2* __restrict__ xy, const int32_t* __restrict__ tri, int64_t V, int64_t T,
    int32_t* __restrict__ origin, hid* __restrict__ twin, hid* __restrict__ next, uint8_t* __restrict__ lcode,
    uint32_t* __restrict__ F0, int64_t bv_stride, uint32_t* __restrict__ C,
    uint8_t* __restrict__ len, int32_t* __restrict__ wlen, unsigned long long* __restrict__ left_key,
    hid* __restrict__ left_e, hid* __restrict__ def_e, uint32_t* __restrict__ SDB,
    int32_t* __restrict__ cnt_ld, DevCounters* ctr, int64_t tile, int64_t tile_next) {
  int32_t* tri_q = reinterpret_cast<int32_t*>(smem_tile);
  int4* tri_q4 = reinterpret_cast<int4*>(smem_tile);
  int16_t* tw_s = reinterpret_cast<int16_t*>(smem_tile + kOffTw);
  uint16_t* slot = reinterpret_cast<uint16_t*>(smem_tile + kOffSlot);
  uint8_t* lc_s = smem_tile + kOffLc;
  // six word arrays in a row (word wl of array r at Sw + r * kTileWords + wl)
  uint32_t* Sw = reinterpret_cast<uint32_t*>(smem_tile + kOffWords);   // seed bits (e order)
  uint32_t* Cw = Sw + kTileWords;                                                // canonical seed bits
  int32_t* Wl = reinterpret_cast<int32_t*>(Cw + kTileWords);                     // loop lengths per C word
  uint32_t* Lm = reinterpret_cast<uint32_t*>(Wl + kTileWords);                   // leftover bits
  uint32_t* Dm = Lm + kTileWords;                                                // deferred bits
  uint32_t* SDm = Dm + kTileWords;                                               // deferred seed bits
  uint32_t* Fw = SDm + kTileWords;                                               // (grid) frontier bits
  uint32_t* Tw = Fw + kTileWords;                                                // (grid) barrier-tip bits
  // overlays of the slot area (after P2)
  uint16_t* succ = slot;

  constexpr bool GRID = MODE == kTileGrid;      // 16 x 128 patches of a row-major list
  constexpr bool SORTED = MODE == kTileSorted;  // runs of the Morton-sorted order perm[]
  constexpr bool SCAT = MODE != kTileContig;    // outputs not one aligned range: words OR-ed
  const TileGeom tg_ = GRID ? tile_geom(tl, T, tile) : contig_geom(T, tile);
  const int64_t f0 = tg_.base;                // global triangle of local triangle 0
  const int64_t seg0 = tg_.seg;               // the tile's list segment
  const int nt = FULL ? kTileTris : GRID ? kTileTris : tg_.nrows;  // (grid: presence per triangle)
  const int g_rows = GRID ? tg_.nrows : 0, g_cols = GRID ? tg_.ncols : 0;
  const int nhe = 3 * nt;
  const int64_t e0 = 3 * f0;
  const int tid = threadIdx.x, lane = tid & 31;
  // local -> global: triangle, half-edge of a quad (grid tiles: rows of 128 triangles R apart)
  auto gtri = [&](int t) -> int64_t {
    return GRID ? f0 + (int64_t)(t >> kGridTWShift) * tl.R + (t & (kGridTW - 1))
                : SORTED ? (int64_t)__ldg(tl.perm + f0 + t) : f0 + t;
  };
  auto ghe = [&](int q) -> int64_t { return SCAT ? 3 * gtri(q >> 2) + (q & 3) : e0 + j_of(q); };
  auto here = [&](int t) -> bool { return FULL || (GRID ? ((t & (kGridTW - 1)) < g_cols && (t >> kGridTWShift) < g_rows) : t < nt); };
#ifdef POLYLLA_PHASE_TIMING
  long long t_phase_ = clock64();
#endif

  // ---- P0: clear the hash slots and the twins (the claims of P1 need the barrier); P1
  // reads the raw triangles straight from global memory (the tile was bulk-prefetched
  // into L2 by the CTA before; staging it in shared memory first measured 1% slower)
  const int32_t* raw = tri + e0;  // (contiguous tiles)
  for (int i = tid; i < kTileSlots / 8; i += kTileThreads)
    reinterpret_cast<uint4*>(slot)[i] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  // (32-bit stores: with 16-byte ones here ptxas 12.9 scheduled the slot clear above's
  // single predicated STS.128 of a partial tile before three of its four source registers
  // were set whenever the table had < 768 uint4s -- garbage slots, caught by the 4,104-slot
  // test variant; the 32-bit form is correct in every variant)
  for (int i = tid; i < kTileQ / 2; i += kTileThreads) reinterpret_cast<uint32_t*>(tw_s)[i] = 0xFFFFFFFFu;
  const TileGeom tn_ = tile_next < 0 ? TileGeom{0, 0, 0, 0} : GRID ? tile_geom(tl, T, tile_next) : contig_geom(T, tile_next);
  const int64_t f0n = tn_.base;  // this CTA's next tile (prefetched), if tile_next >= 0
  if (!SORTED && tile_next >= 0 && (GRID ? tid < tn_.nrows : tid == 0)) {  // the next tile's triangles -> L2 (TMA bulk prefetch)
    const int64_t nn = GRID ? tn_.ncols : (T - f0n < kTileTris ? T - f0n : kTileTris);
    const int32_t* pn = tri + 3 * (f0n + (GRID ? tid * tl.R : 0));  // (grid: one row per thread)
    const uint32_t bytes = (uint32_t)((3 * nn * 4) & ~int64_t(15));
    if (bytes && (reinterpret_cast<uintptr_t>(pn) & 15) == 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pn), "r"(bytes));
  }
  // the raw triangles of this thread, loaded before the barrier
  int32_t ids[kTriIters][3];
#pragma unroll
  for (int i = 0; i < kTriIters; ++i) {
    const int t = tid + i * kTileThreads;
    if (tri_here<FULL, GRID>(i, t, nt, g_rows, g_cols)) {
      const int32_t* rt = SCAT ? tri + 3 * gtri(t) : raw + 3 * t;
      ids[i][0] = rt[0]; ids[i][1] = rt[1]; ids[i][2] = rt[2];
    } else {
      ids[i][0] = ids[i][1] = ids[i][2] = 0;
    }
  }
  __syncthreads();
  PHASE_MARK(0);

  // ---- P1: per triangle: checks, orientation, Lcode; the lo->hi halves claim their home
  // slot of the tile hash with a plain store (last writer wins; P2 verifies)
  const uint64_t pol = policy_evict_last();
  uint32_t bad = 0;
  int flips = 0;
  // the FP64 decisions (R11: IEEE RN, no FMA)
  auto orient_tri = [&](int t, int32_t a, int32_t b, int32_t c) {
    if ((uint64_t)a >= (uint64_t)V || (uint64_t)b >= (uint64_t)V || (uint64_t)c >= (uint64_t)V) {
      bad |= ST_DANGLING;
      a = 0; b = 0; c = 0;
    }
    double2 pa = ld_xy(xy + a, pol), pb = ld_xy(xy + b, pol), pc = ld_xy(xy + c, pol);
    // signed area (x_b-x_a)(y_c-y_a) - (y_b-y_a)(x_c-x_a)
    const double area = __dsub_rn(__dmul_rn(__dsub_rn(pb.x, pa.x), __dsub_rn(pc.y, pa.y)),
                                  __dmul_rn(__dsub_rn(pb.y, pa.y), __dsub_rn(pc.x, pa.x)));
    if (area == 0.0 || a == b || b == c || a == c) bad |= ST_DEGENERATE;
    if (area < 0.0) {
      const int32_t ti = b; b = c; c = ti;
      const double2 tp = pb; pb = pc; pc = tp;
      ++flips;
    }
    const double d0 = sq_len(pa, pb), d1 = sq_len(pb, pc), d2 = sq_len(pc, pa);
    int k = 0;
    double dk = d0;
    if (d1 > dk) { k = 1; dk = d1; }
    if (d2 > dk) { k = 2; }
    lc_s[t] = (uint8_t)k;
    lcode[gtri(t)] = (uint8_t)k;
    tri_q4[t] = make_int4(a, b, c, a);
    if (a < b) st_relaxed16(slot + tile_pos(a, b), 4 * t);
    if (b < c) st_relaxed16(slot + tile_pos(b, c), 4 * t + 1);
    if (c < a) st_relaxed16(slot + tile_pos(c, a), 4 * t + 2);
  };
#pragma unroll
  for (int i = 0; i < kTriIters; ++i) {
    const int t = tid + i * kTileThreads;
    if (!tri_here<FULL, GRID>(i, t, nt, g_rows, g_cols)) continue;
    orient_tri(t, ids[i][0], ids[i][1], ids[i][2]);
  }
  flips = __reduce_add_sync(0xffffffffu, flips);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0) {
    if (flips) atomicAdd(&ctr->n_flips, flips);
    if (bad) raise_status(ctr, bad);
  }
  __syncthreads();
  PHASE_MARK(1);

  // L2 prefetch of the coordinates of the next tile's vertices (its triangles were
  // bulk-prefetched in P0), so that tile's P1 gathers hit L2 instead of HBM: one triangle
  // per thread per pass (P2, P2c, P3), its ids loaded at the start of the pass and the
  // prefetches issued at its end (the loads' latency hides behind the pass)
  const int64_t nn_pf = tile_next >= 0 ? (GRID ? kTileTris : (T - f0n < kTileTris ? T - f0n : kTileTris)) : 0;
  int32_t pf_v[3];
  bool pf_ok = false;
  auto pf_load = [&](int i) {
    const int t = tid + i * kTileThreads;
    pf_ok = t < nn_pf && (!GRID || ((t & (kGridTW - 1)) < tn_.ncols && (t >> kGridTWShift) < tn_.nrows));
    if (pf_ok) {  // volatile: issued here, not sunk next to their use at the end of the pass
      const int32_t* src = tri + 3 * (GRID ? f0n + (int64_t)(t >> kGridTWShift) * tl.R + (t & (kGridTW - 1))
                                           : SORTED ? (int64_t)__ldg(tl.perm + f0n + t) : f0n + t);
      asm volatile("ld.global.nc.b32 %0, [%3];\n\tld.global.nc.b32 %1, [%3+4];\n\tld.global.nc.b32 %2, [%3+8];"
                   : "=r"(pf_v[0]), "=r"(pf_v[1]), "=r"(pf_v[2]) : "l"(src));
    }
  };
  auto pf_issue = [&]() {
    if (pf_ok) {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if ((uint64_t)pf_v[k] < (uint64_t)V) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(xy + pf_v[k]));
    }
  };

  // ---- P2: every half-edge re-reads its home slot (the claims are final: a slot, once
  // claimed, never changes).  lo->hi: the losers of their home slot insert with CAS +
  // linear probing (after the loop, one merged loop per lane).  hi->lo: a twin found in
  // the home slot is recorded now; a different key there -> probed in P2c (after every
  // loser is in); an empty home slot -> no twin in the tile (a loser never lands in an
  // empty home of a key whose lo->hi half exists: that half claimed it).
  pf_load(0);
  uint32_t nm = 0, pend_look = 0;
  {
    uint32_t pend_ins = 0;
#pragma unroll
    for (int i = 0; i < kTriIters; ++i) {
      const int t = tid + i * kTileThreads;
      if (!tri_here<FULL, GRID>(i, t, nt, g_rows, g_cols)) continue;
      const int4 v = tri_q4[t];
      const int32_t vs[4] = {v.x, v.y, v.z, v.w};
      // the three home slots, then the candidates' vertices, then the decisions (loads
      // issued together, predicated, no branch between them)
      uint32_t w[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint32_t o = (uint32_t)vs[k], tg = (uint32_t)vs[k + 1];
        w[k] = ld_relaxed16(slot + tile_pos(min(o, tg), max(o, tg)));
      }
      int32_t ca[3], cb[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const bool look = vs[k] > vs[k + 1] && w[k] != kEmpty16;
        ca[k] = look ? tri_q[w[k]] : -1;
        cb[k] = look ? tri_q[w[k] + 1] : -1;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {  // (flag arithmetic and predicated stores: no divergent branch)
        const int32_t q = 4 * t + k;
        const bool look = vs[k] > vs[k + 1] && w[k] != kEmpty16;
        const bool match = ca[k] == vs[k + 1] && cb[k] == vs[k];  // (ca = -1 unless look)
        pend_ins |= (uint32_t)(vs[k] < vs[k + 1] && w[k] != (uint32_t)q) << (4 * i + k);
        pend_look |= (uint32_t)(look && !match) << (4 * i + k);
        if (match) {
          tw_s[q] = (int16_t)w[k];
          tw_s[w[k]] = (int16_t)q;
        }
      }
    }
    while (pend_ins) {
      const int b = __ffs(pend_ins) - 1;
      pend_ins &= pend_ins - 1;
      const int q = 4 * (tid + (b >> 2) * kTileThreads) + (b & 3);
      nm |= tile_insert_probe(slot, tri_q, q, (uint32_t)tri_q[q], (uint32_t)tri_q[q + 1]);
    }
  }
  pf_issue();
  __syncthreads();
  // ---- P2c: the hi->lo halves whose home slot held another key probe on
  pf_load(1);
  while (pend_look) {
    const int b = __ffs(pend_look) - 1;
    pend_look &= pend_look - 1;
    const int q = 4 * (tid + (b >> 2) * kTileThreads) + (b & 3);
    const int32_t sq = tile_lookup_probe(slot, tri_q, (uint32_t)tri_q[q + 1], (uint32_t)tri_q[q]);
    if (sq >= 0) {
      tw_s[q] = (int16_t)sq;
      tw_s[sq] = (int16_t)q;
    }
  }
  pf_issue();
  if (nm) raise_status(ctr, nm);
  __syncthreads();
  PHASE_MARK(2);

  // ---- P3..P4b run per triangle (thread t = tid + 768 i takes the quad 4t..4t+3: one
  // 8-byte shared access per array instead of three, and the three half-edges' gathers
  // issued together).  A warp's 32 triangles are the 96 half-edges of 3 bit-vector words
  // (tile words 72 i + 3 warp + m, m < 3): per-lane flag bits go to the words by one
  // shuffle + one ballot per word and flag (word_bits below).
  // Loop over every triangle slot of the tile (warp-uniform; triangles past nt of a
  // partial tile contribute zero bits, so every shared word is written).
  static_assert(kTileThreads % 32 == 0 && (kTileTris - (kTriIters - 1) * kTileThreads) % 32 == 0, "uniform");
  const int wl_warp = 3 * (tid >> 5);  // + (3 * 768 / 32) i: tile-local word of the warp's first half-edge
  const int lane_m = lane % 3, lane_ty = lane / 3;  // word stores: lane = 3 * type + m
  // bit k (k < 3) of field f of lane src -> bit `lane` of word m: half-edge h = 32 m + lane
  // of the warp's 96 is half-edge k = h % 3 of the warp's triangle h / 3
  auto word_bits = [&](uint32_t packed, int m, int field) -> uint32_t {
    const int h = 32 * m + lane, src = (h * 0x5556) >> 16, k = h - 3 * src;
    const uint32_t v = __shfl_sync(0xffffffffu, packed, src);
    return __ballot_sync(0xffffffffu, (v >> (4 * field + k)) & 1u);
  };
  auto pick_m = [&](uint32_t w0, uint32_t w1, uint32_t w2) { return lane_m == 0 ? w0 : lane_m == 1 ? w1 : w2; };

  // ---- P3 (per half-edge, e order): origin/twin out (coalesced); rotation successors:
  //   succ[x] = x | FRONT   if x is a frontier half-edge (walk ends there)
  //   succ[x] = x | UNKNOWN if twin(x) is outside the tile (walk must be deferred)
  //   succ[x] = next_q(twin x)  otherwise (cross the non-frontier edge: sweep_out)
  // seed bits S (Alg. 9: a terminal edge's smaller half; never a frontier half-edge, so
  // never deferred) and leftover bits (twin outside the tile) by warp ballots -> Sw / S / Lm
  // (slot 3 of every quad: 0xFFFF, terminal, never a target)
  if (kTriIters > 2) pf_load(2);
  nm = 0;
  for (int i = tid; i < kTileTris; i += kTileThreads) succ[4 * i + 3] = 0xFFFFu;
  {
    // the two ballot words of every iteration are kept by one lane each and stored after
    // the loop (one store per lane instead of a divergent store branch per iteration)
    constexpr bool kBatchWords = kHeIters <= 8;
    const int keep_i = lane & 7;
    const bool keep_l = (lane >> 3) == 1;
    uint32_t kept = 0;
    (void)keep_i; (void)keep_l; (void)kept;
    uint32_t* const s_dst = kBatchWords ? (lane < 8 ? Sw : Lm) : (lane == 0 ? Sw : Lm);
    int q = q_of(tid);
#pragma unroll 4
    for (int i = 0; i < kHeIters; ++i, q = q_step(q)) {
      const int j = tid + i * kTileThreads;
      if (kHePartial && j - lane >= kTileHE) break;  // (warp-uniform)
      bool sd = false, left = false;
      if (FULL || (GRID ? here(q >> 2) : j < nhe)) {
        const int k = q & 3, t = q >> 2;
        // loads issued together: own twin / vertex / Lcode, then the twin's back-pointer and Lcode
        const int32_t tq = tw_s[q];
        const int32_t org = tri_q[q];
        const int32_t lq = lc_s[t];
        const int32_t tqs = tq < 0 ? q : tq;
        const int32_t back = tw_s[tqs];
        const int32_t lt = lc_s[tqs >> 2];
        if (tq >= 0 && back != q) nm = ST_NONMANIFOLD_EDGE;  // twin claimed twice (edge in > 2 triangles)
        if (SCAT) {
          const int64_t ge = ghe(q);
          __stcs(origin + ge, org);
          __stcs(twin + ge, tq >= 0 ? (hid)ghe(tq) : kNoHe);
        } else {
          __stcs(origin + e0 + j, org);
          __stcs(twin + e0 + j, tq >= 0 ? (hid)(e0 + j_of(tq)) : kNoHe);
        }
        const bool front = lq != k && lt != (tq & 3);  // neither half the longest edge of its triangle
        succ[q] = (uint16_t)(tq < 0 ? (q | kSuccUnknown) : front ? (q | kSuccFront) : next_q(tq));
        sd = tq >= 0 && lq == k && lt == (tq & 3);  // terminal edge: the smaller id of the pair (R8)
        if (SORTED) sd = sd && ghe(q) < ghe(tq);     // (sorted tiles: local order is not the id order)
        else sd = sd && q < tq;
        left = tq < 0;
      }
      const uint32_t sw = __ballot_sync(0xffffffffu, sd), lw = __ballot_sync(0xffffffffu, left);
      if constexpr (kBatchWords) {
        if (i == keep_i) kept = keep_l ? lw : sw;  // (stored once, after the loop)
      } else {
        const int wl = (j - lane) >> 5;  // tile-local word of this warp
        // lane 0: Sw, lane 1: Lm (shared); lane 2: the global S
        if (lane < 2) {
          s_dst[wl] = lane == 0 ? sw : lw;
        } else if (!SCAT && lane == 2 && (FULL || j - lane < nhe)) {  // (grid / sorted tiles: flushed at the end)
          F0[2 * bv_stride + (e0 >> 5) + wl] = sw;
        }
      }
    }
    if constexpr (kBatchWords) {  // lanes 0-7: Sw, 8-15: Lm (shared), 16-23: the global S of iteration lane % 8
      const int wl = (tid >> 5) + keep_i * (kTileThreads / 32);
      if (lane < 24 && keep_i < kHeIters && wl < kTileWords) {
        if (lane < 16) s_dst[wl] = kept;
        else if (!SCAT && (FULL || 32 * wl < nhe)) F0[2 * bv_stride + (e0 >> 5) + wl] = kept;
      }
    }
  }
  if (kTriIters > 2) pf_issue();
  if (nm) raise_status(ctr, nm);
  uint32_t* const seed_n = reinterpret_cast<uint32_t*>(smem_tile + kOffWords + kWordBytes);  // (dead table space)
  uint16_t* const seed_list = reinterpret_cast<uint16_t*>(seed_n + 4);
  if (POLYLLA_P6_LIST && tid == 0) *seed_n = 0;
  __syncthreads();
  PHASE_MARK(3);

  // ---- P4a: pointer jumping in place: each round doubles the resolved chain length.  A
  // successor read while its owner rewrites it is the old or the new value, both on the
  // chain and at least as far along as the round before, so after r rounds every entry is
  // >= 2^r steps ahead (or terminal); further along only moves work from the global fixup
  // into the tile, which computes the same next.  (Slot 3 of a quad: 0xFFFF, terminal.)
  static_assert(kTileJumps <= 4, "pointer-jumping rounds");
#pragma unroll 1
  for (int round = 0; round < kTileJumps; ++round) {
#pragma unroll
    for (int i = 0; i < kTriIters; ++i) {
      const int t = tid + i * kTileThreads;
      if (!tri_here<FULL, GRID>(i, t, nt, g_rows, g_cols)) continue;
      const uint2 s2 = *reinterpret_cast<const uint2*>(succ + 4 * t);  // (own quad: only this thread writes it)
      const uint32_t sc[3] = {s2.x & 0xFFFFu, s2.x >> 16, s2.y & 0xFFFFu};
      uint32_t d[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) d[k] = (sc[k] & (kSuccFront | kSuccUnknown)) ? sc[k] : ld_relaxed16(succ + sc[k]);
      *reinterpret_cast<uint2*>(succ + 4 * t) = make_uint2(d[0] | (d[1] << 16), d[2] | 0xFFFF0000u);
    }
    __syncthreads();
  }
  PHASE_MARK(4);

  // ---- P4b: per triangle: next (Alg. 11) of its three half-edges, F words (Alg. 8), tips
  // (next == twin, R4), deferred half-edges; the local next in quad indices (nx_q; the
  // global origin/twin/next are written from the quad arrays in half-edge order in P5)
  int16_t* nx_q = tw_s;  // quad-indexed local next over the twins (each thread reads its quad's twins first)
  // the 9 words of iteration i (3 words x frontier / tip / deferred) are kept by lanes
  // 9i .. 9i + 8 and stored once after the loop (POLYLLA_P4B_BATCH)
#ifndef POLYLLA_P4B_BATCH
#define POLYLLA_P4B_BATCH 1
#endif
  constexpr bool kBatch4 = POLYLLA_P4B_BATCH && 9 * kTriIters <= 32;
#if POLYLLA_P6_LIST
  if (tid < kTileWords) {  // the tile's seeds (S bits, final since P3) listed for P6 (one seed per thread there)
    uint32_t sb = Sw[tid];
    const int c = __popc(sb);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += a;
    }
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(seed_n, (uint32_t)incl);
    base = __shfl_sync(0xffffffffu, base, 31) + (uint32_t)(incl - c);
    for (; sb; sb &= sb - 1) seed_list[base++] = (uint16_t)(tid * 32 + __ffs(sb) - 1);
  }
#endif
  const int my_it = lane / 9, my_f = (lane % 9) / 3;
  uint32_t kept4 = 0;
  (void)my_it; (void)my_f; (void)kept4;
  if constexpr (kBatch4) {  // (Cw, Wl, SDm: zero before P6's atomics)
    for (int w = tid; w < kTileWords; w += kTileThreads) {
      Sw[kTileWords + w] = 0u;
      Sw[2 * kTileWords + w] = 0u;
      Sw[5 * kTileWords + w] = 0u;
    }
  }
#pragma unroll
  for (int i = 0; i < kTriIters; ++i) {
    if (!(i < kTriIters - 1 || tid < kTileTris - (kTriIters - 1) * kTileThreads)) continue;
    const int t = tid + i * kTileThreads;
    uint32_t packed = 0;  // field 0: frontier, 1: tip, 2: deferred
    if (here(t)) {
      const uint2 s2 = *reinterpret_cast<const uint2*>(succ + 4 * t);
      const uint2 tw2 = *reinterpret_cast<const uint2*>(tw_s + 4 * t);
      const uint32_t sc[3] = {s2.x & 0xFFFFu, s2.x >> 16, s2.y & 0xFFFFu};
      const int32_t tq[3] = {(int16_t)(tw2.x & 0xFFFFu), (int16_t)(tw2.x >> 16), (int16_t)(tw2.y & 0xFFFFu)};
      int32_t nl[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int32_t q = 4 * t + k;
        const bool left = sc[k] == (uint32_t)(q | kSuccUnknown);
        bool fr = sc[k] == (uint32_t)(q | kSuccFront);  // terminal of its own chain: a frontier half-edge
        bool tip = false, deferred = left;
        int32_t nx = next_q(q);
        if (fr) {
          uint32_t r = sc[k == 2 ? 0 : k + 1];  // succ[next_q(q)]: first frontier half-edge about target, if reached
          for (int h = 0; h < kTileHops && !(r & (kSuccFront | kSuccUnknown)); ++h) r = succ[r];
          if (r & kSuccFront) {
            nx = (int32_t)(r & kSuccIdx);
            tip = nx == tq[k];  // barrier tip: next == twin (R4)
          } else {
            deferred = true;
            fr = false;  // the fixup sets every bit of a deferred half-edge
          }
        }
        nl[k] = deferred ? -1 : tip ? (kNxTip | tq[k]) : nx;  // a barrier tip (its loop is split by the repair)
        packed |= ((uint32_t)fr << k) | ((uint32_t)tip << (4 + k)) | ((uint32_t)deferred << (8 + k));
      }
      *reinterpret_cast<uint2*>(nx_q + 4 * t) =
          make_uint2((uint32_t)(uint16_t)nl[0] | ((uint32_t)(uint16_t)nl[1] << 16), (uint32_t)(uint16_t)nl[2] | 0xFFFF0000u);
    }
    const int wl0 = (3 * kTileThreads / 32) * i + wl_warp;
    const uint32_t f0w = word_bits(packed, 0, 0), f1w = word_bits(packed, 1, 0), f2w = word_bits(packed, 2, 0);
    const uint32_t t0w = word_bits(packed, 0, 1), t1w = word_bits(packed, 1, 1), t2w = word_bits(packed, 2, 1);
    const uint32_t d0w = word_bits(packed, 0, 2), d1w = word_bits(packed, 1, 2), d2w = word_bits(packed, 2, 2);
    if constexpr (kBatch4) {
      if (my_it == i)
        kept4 = my_f == 0 ? pick_m(f0w, f1w, f2w) : my_f == 1 ? pick_m(t0w, t1w, t2w) : pick_m(d0w, d1w, d2w);
      continue;
    }
    // lanes 0-11: shared Cw (0), Wl (0), Dm, SDm (0); lanes 12-20: global F0, F1, TB
    if (lane < 12) {
      const int r = lane_ty == 0 ? 1 : lane_ty == 1 ? 2 : lane_ty == 2 ? 4 : 5;  // Cw, Wl, Dm, SDm
      Sw[r * kTileWords + wl0 + lane_m] = lane_ty == 2 ? pick_m(d0w, d1w, d2w) : 0u;
    } else if (SCAT) {  // the frontier and tip words, flushed at the end
      if (lane < 15) Fw[wl0 + lane_m] = pick_m(f0w, f1w, f2w);
      else if (lane >= 18 && lane < 21) Tw[wl0 + lane_m] = pick_m(t0w, t1w, t2w);
    } else if (lane < 21 && (FULL || 32 * (wl0 + lane_m) < nhe)) {
      const int g = lane_ty == 4 ? 0 : lane_ty == 5 ? 1 : 3;  // F0, F1, TB
      F0[g * bv_stride + (e0 >> 5) + wl0 + lane_m] = lane_ty == 6 ? pick_m(t0w, t1w, t2w) : pick_m(f0w, f1w, f2w);
    }
  }
  if constexpr (kBatch4) {
    const int wl = (3 * kTileThreads / 32) * my_it + wl_warp + lane_m;
    if (lane < 9 * kTriIters && wl < kTileWords) {
      if (my_f == 2) Dm[wl] = kept4;
      else if (SCAT) (my_f == 0 ? Fw : Tw)[wl] = kept4;  // (flushed at the end)
      else if (FULL || 32 * wl < nhe) {
        if (my_f == 0) {
          F0[(e0 >> 5) + wl] = kept4;
          F0[bv_stride + (e0 >> 5) + wl] = kept4;
        } else {
          F0[3 * bv_stride + (e0 >> 5) + wl] = kept4;
        }
      }
    }
  }
  __syncthreads();
  PHASE_MARK(5);

  // ---- P5: the leftover (key, id) and deferred lists as per-tile segments at e0 of
  // left_e/left_key/def_e (counts in cnt_ld[2 * tile + {0, 1}]), one word per thread of
  // warps 0-5: a word's exclusive prefix is the warp's shuffle scan plus the popcounts of
  // the earlier warps' words, which every lane sums itself (no barrier, no global atomic)
  if (tid < kTileWords) {
    uint32_t lw = Lm[tid], dw = Dm[tid];
    const int cl = __popc(lw), cd = __popc(dw);
    int il = cl, id = cd;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, il, o), b = __shfl_up_sync(0xffffffffu, id, o);
      if (lane >= o) { il += a; id += b; }
    }
    int bl = 0, bd = 0;
    for (int w = lane; w < (tid & ~31); w += 32) { bl += __popc(Lm[w]); bd += __popc(Dm[w]); }
    bl = __reduce_add_sync(0xffffffffu, bl);
    bd = __reduce_add_sync(0xffffffffu, bd);
    if (tid == kTileWords - 1) {
      reinterpret_cast<int2*>(cnt_ld)[tile] = make_int2(bl + il, bd + id);
      if (bl + il) atomicAdd(&ctr->n_left, bl + il);  // totals (result unused: a reduction)
      if (bd + id) atomicAdd(&ctr->n_def, bd + id);
    }
    int64_t pl = seg0 + bl + il - cl, pd = seg0 + bd + id - cd;
    while (lw) {
      const int j = tid * 32 + __ffs(lw) - 1;
      lw &= lw - 1;
      const int q = q_of(j);
      const int32_t o = tri_q[q], tg = tri_q[q + 1];
      const uint64_t lo = (uint32_t)min(o, tg), hi = (uint32_t)max(o, tg);
      left_key[pl] = (lo << 32) | hi | (o > tg ? kLeftDown : 0ull);  // undirected key + direction bit
      left_e[pl++] = (hid)(SCAT ? ghe(q) : e0 + j);
    }
    while (dw) {
      const int j = tid * 32 + __ffs(dw) - 1;
      def_e[pd++] = (hid)(SCAT ? ghe(q_of(j)) : e0 + j);
      dw &= dw - 1;
    }
  }

  // ---- P5b: next out in half-edge order (coalesced stores; a per-triangle store of three
  // consecutive ids writes a third of 12 sectors per instruction): nx_q's resolved
  // successor, twin for a barrier tip, untouched for a deferred half-edge
  {
    int q = q_of(tid);
#pragma unroll 4
    for (int i = 0; i < kHeIters; ++i, q = q_step(q)) {
      const int j = tid + i * kTileThreads;
      if (SCAT) {
        if (j >= kTileHE) break;
        if (!here(q >> 2)) continue;
        const int32_t nl = nx_q[q];
        if (nl != -1) __stcs(next + ghe(q), (hid)ghe(nl & ~kNxTip));
        continue;
      }
      if ((!FULL || kHePartial) && j >= nhe) break;
      const int32_t nl = nx_q[q];
      if (nl != -1) __stcs(next + e0 + j, (hid)(e0 + j_of(nl & ~kNxTip)));
    }
  }

  // ---- P6: seeds whose polygon closes inside the tile (Alg. 12 + Overwrite seeds,
  // PAPER.md L778-849): land on a frontier half-edge by rotation (the resolved successor
  // chain), walk the loop on nx_q, keep the minimum id and the length.  Loops that touch
  // a deferred half-edge or a barrier tip (repaired later) are handed to the global
  // seed walk (bit-vector SDB).  kSeedLanes threads per word take its seeds in turn.
  {
#if POLYLLA_P6_LIST
    const int n_seeds = (int)*seed_n;  // one listed seed per thread (the walks fill whole warps),
    // the first ones to the threads past warps 0-5, which are still writing P5's lists
    const int s0 = tid >= kTileWords ? tid - kTileWords : tid + (kTileThreads - kTileWords);
    for (int si = s0; si < n_seeds; si += kTileThreads) {
      const int32_t sj = seed_list[si];
#else
    constexpr int kSeedLanes = kTileThreads / kTileWords;  // 4 (the threads past kSeedLanes * 192 idle)
    static_assert(kSeedLanes >= 1, "threads per word");
    const int wsd = tid / kSeedLanes, sub = tid % kSeedLanes;
    uint32_t sb = wsd < kTileWords ? Sw[wsd] : 0u;
    for (int k = 0; k < sub && sb; ++k) sb &= sb - 1;
    while (sb) {
      const int32_t sj = wsd * 32 + __ffs(sb) - 1;
      for (int k = 0; k < kSeedLanes && sb; ++k) sb &= sb - 1;
#endif
      uint16_t r = succ[q_of(sj)];  // the frontier half-edge the rotation reaches, if resolved
      for (int h = 0; h < kTileHops && !(r & (kSuccFront | kSuccUnknown)); ++h) r = succ[r];
      bool ok = (r & kSuccFront) != 0, tipped = false;
      const bool landed = ok;
      int32_t mn = 0, n = 0, x = 0;  // quad indices (the same order as half-edge ids, but for sorted tiles)
      int64_t gmin = INT64_MAX;      // (sorted tiles: the minimum global id)
      if (ok) {
        x = r & kSuccIdx;
        int32_t y = x;
        mn = x;
        do {
          mn = min(mn, y);
          if (SORTED) gmin = min(gmin, ghe(y));
          ++n;
          y = nx_q[y];
          if ((uint32_t)y >= (uint32_t)kNxTip || n > kP6MaxLen) {  // deferred (-1) / barrier tip / long loop
            ok = false;
            tipped = y >= 0 && (y & kNxTip);
            break;
          }
        } while (y != x);
      }
      if (ok && SORTED) {  // canonical seed = the minimum global id: its bit set in the global C directly
        len[gmin] = len_code(n);
        const uint32_t gbit = 1u << (gmin & 31);
        if (!(atomicOr(&C[gmin >> 5], gbit) & gbit)) atomicAdd(&wlen[gmin >> 5], n);  // first setter only
      } else if (ok) {
        const int64_t gmn = ghe(mn);  // (the loop minimum: quad and half-edge orders agree)
        mn = j_of(mn);
        len[gmn] = len_code(n);
        const uint32_t bit = 1u << (mn & 31);
        if (!(atomicOr(&Cw[mn >> 5], bit) & bit)) {  // first setter only
          if (SCAT) atomicAdd(&wlen[gmn >> 5], n);   // (grid / sorted: global words, zeroed before the build)
          else atomicAdd(&Wl[mn >> 5], n);
        }
      } else if (!tipped) {
        // (a loop through a barrier tip is split by the repair, and every piece borders a
        // middle edge whose two halves k_repair_mid seeds: this seed would add nothing).
        // The global walk starts from the frontier half-edge the seed landed on when the
        // landing stayed in the tile (the same loop: F1 adds frontier edges only to
        // repaired loops, whose pieces the middle-edge halves seed anyway), else from the seed.
        const int32_t g = landed ? j_of(x) : sj;
        atomicOr(&SDm[g >> 5], 1u << (g & 31));
      }
    }
  }
  __syncthreads();
  PHASE_MARK(6);
  if (GRID) {
    // local word L = 12 r + m holds half-edges 32 m .. 32 m + 31 of triangle row r (384 per
    // row): global bits 3 (base + r R) + 32 m onward, not word-aligned -> two atomicOr
    // (the global words were zeroed before the build; neighbouring tiles share words)
    if (tid < kTileWords && tid / 12 < g_rows) {
      const int64_t gb = 3 * (f0 + (int64_t)(tid / 12) * tl.R) + 32 * (tid % 12);
      const int64_t gw = gb >> 5;
      const int sh = (int)(gb & 31);
      auto put = [&](uint32_t* base, uint32_t v) {
        if (!v) return;
        atomicOr(base + gw, v << sh);
        if (sh) atomicOr(base + gw + 1, v >> (32 - sh));
      };
      put(F0, Fw[tid]);
      put(F0 + bv_stride, Fw[tid]);
      put(F0 + 2 * bv_stride, Sw[tid]);
      put(F0 + 3 * bv_stride, Tw[tid]);
      put(C, Cw[tid]);
      put(SDB, SDm[tid]);
    }
  } else if (SORTED) {
    // each triangle's three bits go to global bits 3f .. 3f+2 (f = perm[...]): one (or
    // two, across a word boundary) atomicOr per array with any bit set
    for (int u = tid; u < nt; u += kTileThreads) {
      const int64_t gb = 3 * gtri(u);
      const int64_t gw = gb >> 5;
      const int sh = (int)(gb & 31), lj = 3 * u;
      auto bits3 = [&](const uint32_t* w) -> uint32_t {  // local bits lj .. lj+2 (may straddle a word)
        const uint64_t two = (uint64_t)w[lj >> 5] | ((lj >> 5) + 1 < kTileWords ? (uint64_t)w[(lj >> 5) + 1] << 32 : 0);
        return (uint32_t)(two >> (lj & 31)) & 7u;
      };
      auto put = [&](uint32_t* base, uint32_t v) {
        if (!v) return;
        atomicOr(base + gw, v << sh);
        if (sh > 29) atomicOr(base + gw + 1, v >> (32 - sh));
      };
      const uint32_t f = bits3(Fw);
      put(F0, f);
      put(F0 + bv_stride, f);
      put(F0 + 2 * bv_stride, bits3(Sw));
      put(F0 + 3 * bv_stride, bits3(Tw));
      put(SDB, bits3(SDm));  // (C: set directly by P6)
    }
  } else if (tid * 32 < nhe) {
    const int64_t w = (e0 >> 5) + tid;
    C[w] = Cw[tid];
    wlen[w] = Wl[tid];
    SDB[w] = SDm[tid];
  }
  PHASE_MARK(7);
}

// One CTA per tile; while it works it prefetches into L2 the triangles and vertex
// coordinates of the tile that will start when it ends.  Full tiles take the specialised
// body (constant trip counts, no bounds checks), the ragged last tile the generic one.
template <int MODE>
__global__ void __launch_bounds__(kTileThreads, 2)
    k_tile(const double2* __restrict__ xy, const int32_t* __restrict__ tri, int64_t V, int64_t T,
           int32_t* __restrict__ origin, hid* __restrict__ twin, hid* __restrict__ next,
           uint8_t* __restrict__ lcode, uint32_t* __restrict__ F0, int64_t bv_stride, uint32_t* __restrict__ C, uint8_t* __restrict__ len, int32_t* __restrict__ wlen,
           unsigned long long* __restrict__ left_key, hid* __restrict__ left_e, hid* __restrict__ def_e,
           uint32_t* __restrict__ SDB, int32_t* __restrict__ cnt_ld, DevCounters* ctr,
           int64_t prefetch_dist, int64_t tile_base, const Tiling tl) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_tile[];
  const int64_t ntiles = MODE != kTileContig ? tl.ntiles : (T + kTileTris - 1) / kTileTris;
  // tiles [tile_base, tile_base + gridDim.x): all of them, or one chunk of an upload
  // pipeline (polylla_run_host)
  const int64_t tile = tile_base + sched_tile(blockIdx.x, gridDim.x);
  // the tile that starts about when this one ends (blocks are dispatched in index order,
  // kResident at a time): its data is prefetched into L2, which every SM shares
  const int64_t nxt = tile + prefetch_dist < ntiles ? tile + prefetch_dist : -1;
  bool full;
  if (MODE == kTileGrid) {
    const TileGeom g = tile_geom(tl, T, tile);
    full = g.nrows == kGridTH && g.ncols == kGridTW;
  } else {
    full = (tile + 1) * kTileTris <= T;
  }
  if (full)
    tile_body<true, MODE>(smem_tile, tl, xy, tri, V, T, origin, twin, next, lcode, F0, bv_stride, C, len, wlen,
                          left_key, left_e, def_e, SDB, cnt_ld, ctr, tile, nxt);
  else
    tile_body<false, MODE>(smem_tile, tl, xy, tri, V, T, origin, twin, next, lcode, F0, bv_stride, C, len, wlen,
                           left_key, left_e, def_e, SDB, cnt_ld, ctr, tile, nxt);
}

#ifdef POLYLLA_PHASE_TIMING
extern "C" __attribute__((visibility("default"))) int polylla_debug_phase_cycles(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles)) != cudaSuccess) return -1;
  if (reset) {
    static const unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

__device__ __forceinline__ uint64_t hash_cap_for(uint32_t n) {
  uint64_t c = 1024;
  while (c < 2ull * (uint64_t)n) c <<= 1;
  return c;
}

__global__ void k_hash_clear(DevCounters* ctr, uint32_t* ehash, int64_t cap_max, int64_t V, int64_t T) {
  pdl_enter();
  const uint64_t cap = hash_cap_for(ctr->n_left);
  if ((int64_t)cap > cap_max) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_status(ctr, ST_INTERNAL);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr->hash_cap = (uint32_t)cap;
    // locality-preserving homes only where leftovers are dense (>= 1/6 of the half-edges:
    // a mesh whose tiles are thin strips, e.g. row-major grids); sparse leftovers of
    // spatially ordered random meshes keep the mixing hash (measured: config 3 +10% with
    // the locality homes, config 4 -72%, config 5 -40%)
    ctr->hash_scale = 2 * (int64_t)ctr->n_left >= T
                          ? (unsigned long long)(((unsigned __int128)cap << 32) / (unsigned long long)V)
                          : 0ull;
  }
  // cap is a power of two >= 1024 and ehash is 256-B aligned: 16-B stores
  uint4* h4 = reinterpret_cast<uint4*>(ehash);
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap / 4; i += gridDim.x * blockDim.x)
    h4[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
}

// global hash over leftover half-edges: pair the two halves of each cross-tile edge.
// The leftovers of tile t are entries [3 * kTileTris * t, + cnt_ld[2t]) of left_key/left_e;
// one block per tile segment (grid-stride over tiles).
// Dense leftovers take home slots that preserve vertex-id locality: home = lo * cap / V
// (+ 0-3 from hi), so keys of nearby vertices hash to nearby slots.  Where vertex ids follow space (row-major grids,
// configs 4-5, a third of all half-edges crossing tiles) the probes of concurrently
// running tiles stay in a narrow, L2-resident band of the table; spatially random ids
// (configs 2-3) spread uniformly as with a mixing hash.
__device__ __forceinline__ uint32_t left_home(uint32_t lo, uint32_t hi, unsigned long long scale, uint32_t mask) {
  if (!scale) return mix32(lo, hi) & mask;
  return ((uint32_t)(((unsigned long long)lo * scale) >> 32) + ((hi * 0x9E3779B1u) >> 30)) & mask;
}
__global__ void k_left_insert(DevCounters* ctr, int64_t ntiles, int64_t T, const Tiling tl,
                              const int32_t* __restrict__ cnt_ld, unsigned long long* left_key,
                              const hid* __restrict__ left_e, hid* twin, uint32_t* ehash) {
  pdl_enter();
  if (ctr->status) return;
  const uint32_t mask = (uint32_t)ctr->hash_cap - 1;
  const unsigned long long scale = ctr->hash_scale;
  for (int64_t it = blockIdx.x; it < ntiles; it += gridDim.x) {
    const int64_t tile = sched_tile(it, ntiles);
    const int32_t n = cnt_ld[2 * tile];
    const int64_t base = tile_geom(tl, T, tile).seg;
    for (int32_t k = threadIdx.x; k < n; k += blockDim.x) {
      const int64_t i = base + k;  // < 3T <= 2^32 - 2: a slot value never equals kEmpty
      const unsigned long long kd = left_key[i], key = kd & ~kLeftDown;
      const hid ei = left_e[i];
      uint32_t h = left_home((uint32_t)(key >> 32), (uint32_t)key, scale, mask);
      for (uint32_t probe = 0; probe <= mask; ++probe) {
        uint32_t s = ehash[h];
        if (s == kEmpty) {
          const uint32_t old = atomicCAS(&ehash[h], kEmpty, (uint32_t)i);
          if (old == kEmpty) break;
          s = old;
        }
        const unsigned long long sd = left_key[s];
        if ((sd & ~(kLeftDown | kLeftPaired)) == key) {
          // a pair must run in opposite directions; the pairing is claimed on the slot
          // holder's key (bit 31: vertex ids < 2^31), so a third copy finds it taken
          if (((sd ^ kd) & kLeftDown) == 0 || (sd & kLeftPaired) ||
              atomicCAS(left_key + s, sd, sd | kLeftPaired) != sd) {
            raise_status(ctr, ST_NONMANIFOLD_EDGE);
            break;
          }
          const hid es = left_e[s];
          twin[ei] = es;
          twin[es] = ei;
          left_key[i] = kd | kLeftPaired;  // (own entry, never in the hash): both halves flagged for the ranking
          break;
        }
        h = (h + 1) & mask;
      }
    }
  }
}

// Leftovers that found no partner lie on the domain boundary.  Border ids follow R9:
// b = 3T + rank(e) over the unmatched interior half-edges in ascending order.  Each tile
// segment is in ascending e order, so the rank is (border half-edges of the earlier
// tiles) + (rank inside the segment):
//   k_border_rank  one block per tile segment: the unmatched leftovers (no kLeftPaired
//                  flag: the segment's keys are read coalesced instead of a random twin
//                  per leftover) in segment order -> blist, written over the segment's own
//                  dead keys (4-byte entry 2 * base + rank <= the chunk being read), their
//                  count -> bcnt[tile]
//   k_border_scan  one block: exclusive prefix of bcnt over the tiles, B = the total
//   k_border_emit  one block per tile segment: b = 3T + base + rank; twin/origin of b and
//                  vmap[origin(b)] = b (written only at border vertices: never cleared;
//                  k_border_next reads it only at border vertices and verifies it)
constexpr int kSegThreads = 256;

__global__ void __launch_bounds__(kSegThreads)
    k_border_rank(DevCounters* ctr, int64_t ntiles, const int32_t* __restrict__ cnt_ld,
                  const hid* __restrict__ left_e, const unsigned long long* left_key, hid* blist,
                  uint32_t* __restrict__ bcnt) {
  pdl_enter();
  __shared__ int32_t wtot[kSegThreads / 32];
  if (ctr->status) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t it = blockIdx.x; it < ntiles; it += gridDim.x) {
    const int64_t tile = sched_tile(it, ntiles);
    const int32_t n = cnt_ld[2 * tile];
    const int64_t base = 3 * kTileTris * tile;
    int carry = 0;
    for (int32_t k0 = 0; k0 < n; k0 += kSegThreads) {  // block-uniform trip count
      const int32_t k = k0 + threadIdx.x;
      const bool un = k < n && !(left_key[base + k] & kLeftPaired);
      const hid e = un ? left_e[base + k] : kNoHe;
      const uint32_t m = __ballot_sync(0xffffffffu, un);
      if (lane == 0) wtot[wid] = __popc(m);
      __syncthreads();
      int pre = carry, tot = 0;
      for (int w = 0; w < kSegThreads / 32; ++w) {
        if (w < wid) pre += wtot[w];
        tot += wtot[w];
      }
      if (un) blist[2 * base + pre + __popc(m & ((1u << lane) - 1))] = e;  // segment-local rank order
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) bcnt[tile] = (uint32_t)carry;
  }
}

constexpr int kBorderScanThreads = 1024;
__global__ void __launch_bounds__(kBorderScanThreads)
    k_border_scan(DevCounters* ctr, int64_t ntiles, int64_t T3, int64_t Bmax, uint32_t* bcnt) {
  pdl_enter();
  constexpr int NW = kBorderScanThreads / 32;
  __shared__ long long wsum[NW];
  if (ctr->status) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t per = ((ntiles + NW - 1) / NW + 31) & ~int64_t(31);
  const int64_t t0 = wid * per, t1 = t0 + per < ntiles ? t0 + per : ntiles;
  long long sum = 0;
  for (int64_t t = t0 + lane; t < t1; t += 32) sum += bcnt[t];
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) wsum[wid] = sum;
  __syncthreads();
  if (wid == 0) {
    const long long v = wsum[lane];
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    wsum[lane] = inc - v;
    if (lane == 31) {
      if (T3 + inc > kMaxHalfedges) raise_status(ctr, ST_OVERFLOW);
      else if (inc > Bmax) raise_status(ctr, ST_BORDER_CAP);  // nothing is written past 3T + Bmax
      ctr->n_border = (uint32_t)inc;
    }
  }
  __syncthreads();
  long long carry = wsum[wid];
  for (int64_t tb0 = t0; tb0 < t1; tb0 += 32) {
    const int64_t t = tb0 + lane;
    const long long v = t < t1 ? bcnt[t] : 0;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (t < t1) bcnt[t] = (uint32_t)(carry + inc - v);  // in place: the exclusive base of the tile
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

__global__ void __launch_bounds__(kSegThreads)
    k_border_emit(DevCounters* ctr, int64_t ntiles, int64_t T3, const hid* __restrict__ blist,
                  const uint32_t* __restrict__ bbase, int32_t* origin, hid* twin, hid* vmap) {
  pdl_enter();
  if (ctr->status) return;
  const uint32_t nb = ctr->n_border;
  for (int64_t it = blockIdx.x; it < ntiles; it += gridDim.x) {
    const int64_t tile = sched_tile(it, ntiles);
    const uint32_t b0 = bbase[tile];
    const int32_t n = (int32_t)((tile + 1 < ntiles ? bbase[tile + 1] : nb) - b0);
    const int64_t base = 3 * kTileTris * tile;
    for (int32_t k = threadIdx.x; k < n; k += kSegThreads) {
      const hid e = blist[2 * base + k];
      const hid b = (hid)(T3 + b0 + k);
      const int32_t v = origin[next_in(e)];  // origin(b) = target(e)
      twin[e] = b;
      twin[b] = e;
      origin[b] = v;
      vmap[v] = b;
    }
  }
}

// Grid tiling: tile segments are not in ascending half-edge order, so the unmatched
// leftovers are marked in the bit-vector BB (zeroed before the build) and ranked by bit
// order (R9): per chunk of 192 words a popcount (k_bb_count, one warp per chunk), the
// chunks' exclusive prefix (k_border_scan), then each chunk's bits in order (k_bb_emit).
__global__ void k_bb_mark(DevCounters* ctr, int64_t ntiles, int64_t T, const Tiling tl,
                          const int32_t* __restrict__ cnt_ld, const hid* __restrict__ left_e,
                          const unsigned long long* __restrict__ left_key, uint32_t* BB) {
  pdl_enter();
  if (ctr->status) return;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int32_t n = cnt_ld[2 * tile];
    const int64_t base = tile_geom(tl, T, tile).seg;
    for (int32_t k = threadIdx.x; k < n; k += blockDim.x) {
      if (left_key[base + k] & kLeftPaired) continue;  // (paired: flagged by k_left_insert)
      const hid e = left_e[base + k];
      atomicOr(&BB[e >> 5], 1u << (e & 31));
    }
  }
}

constexpr int kBBChunk = 192;  // words per chunk (6 per lane)
__global__ void k_bb_count(DevCounters* ctr, int64_t n_words, int64_t nchunks, const uint32_t* __restrict__ BB,
                           uint32_t* __restrict__ bcnt) {
  pdl_enter();
  if (ctr->status) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunks; ch += nw) {
    int c = 0;
    for (int k = lane; k < kBBChunk; k += 32) {
      const int64_t w = ch * kBBChunk + k;
      if (w < n_words) c += __popc(BB[w]);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) bcnt[ch] = (uint32_t)c;
  }
}

__global__ void k_bb_emit(DevCounters* ctr, int64_t n_words, int64_t nchunks, int64_t T3,
                          const uint32_t* __restrict__ BB, const uint32_t* __restrict__ bbase, int32_t* origin,
                          hid* twin, hid* vmap) {
  pdl_enter();
  if (ctr->status) return;
  const int lane = threadIdx.x & 31;
  constexpr int kWPL = kBBChunk / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunks; ch += nw) {
    uint32_t bw[kWPL];
    int c = 0;
#pragma unroll
    for (int k = 0; k < kWPL; ++k) {
      const int64_t w = ch * kBBChunk + kWPL * lane + k;
      bw[k] = w < n_words ? BB[w] : 0u;
      c += __popc(bw[k]);
    }
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    uint32_t r = bbase[ch] + (uint32_t)(inc - c);
#pragma unroll
    for (int k = 0; k < kWPL; ++k) {
      const int64_t w = ch * kBBChunk + kWPL * lane + k;
      for (uint32_t b = bw[k]; b; b &= b - 1, ++r) {
        const hid e = (hid)(w * 32 + __ffs(b) - 1);
        const hid bh = (hid)(T3 + r);
        const int32_t v = origin[next_in(e)];  // origin(b) = target(e)
        twin[e] = bh;
        twin[bh] = e;
        origin[bh] = v;
        vmap[v] = bh;
      }
    }
  }
}

// next(b) = the border half-edge whose origin is target(b) = origin(twin(b)).  A vertex
// with two outgoing border half-edges keeps only one of them in vmap: the other fails
// the vmap[origin(b)] == b check (NON_MANIFOLD_VERTEX).
__global__ void k_border_next(DevCounters* ctr, int64_t T3, const int32_t* __restrict__ origin,
                              const hid* __restrict__ twin, const hid* __restrict__ vmap, hid* next) {
  pdl_enter();
  if (ctr->status) return;
  const uint32_t nb = ctr->n_border;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const hid b = (hid)(T3 + i);
    const int32_t v = origin[twin[b]];
    const hid nx = vmap[v];
    const bool ok = vmap[origin[b]] == b && nx >= T3 && nx - T3 < nb && origin[nx] == v;
    if (!ok) raise_status(ctr, ST_NONMANIFOLD_VERTEX);
    next[b] = ok ? nx : kNoHe;
  }
}

// ---- the sorted tiling (POLYLLA_BUILD_SORT): a counting sort of the triangles by the
// Morton cell (8 bits per axis) of their first vertex in the bounding box of the vertices
// (one coordinate gather per triangle; any point of the triangle groups as well).
// Only the grouping into tiles depends on it (every output is the same bits for any
// order), so ties within a cell are left in atomic order.
__device__ __forceinline__ unsigned long long ord_of(double d) {  // order-preserving uint64 of a double
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double of_ord(unsigned long long o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o));
}
__global__ void k_sort_init(unsigned long long* bbox, uint32_t* hist, int64_t cells) {
  pdl_enter();
  if (blockIdx.x == 0 && threadIdx.x < 4) bbox[threadIdx.x] = (threadIdx.x & 1) ? 0ull : ~0ull;  // min x, max x, min y, max y
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += (int64_t)gridDim.x * blockDim.x)
    hist[i] = 0;
}
__global__ void __launch_bounds__(256) k_sort_bbox(const double2* __restrict__ xy, int64_t V, unsigned long long* bbox) {
  pdl_enter();
  __shared__ unsigned long long red[4][8];
  unsigned long long mnx = ~0ull, mxx = 0, mny = ~0ull, mxy = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = xy[i];
    const unsigned long long ox = ord_of(p.x), oy = ord_of(p.y);
    mnx = min(mnx, ox); mxx = max(mxx, ox); mny = min(mny, oy); mxy = max(mxy, oy);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = mnx; red[1][w] = mxx; red[2][w] = mny; red[3][w] = mxy; }
  __syncthreads();
  if (threadIdx.x == 0) {  // one atomic per block and bound (warp-level atomics serialised on 4 words)
    for (int k = 1; k < 8; ++k) {
      mnx = min(mnx, red[0][k]); mxx = max(mxx, red[1][k]); mny = min(mny, red[2][k]); mxy = max(mxy, red[3][k]);
    }
    atomicMin(bbox, mnx); atomicMax(bbox + 1, mxx); atomicMin(bbox + 2, mny); atomicMax(bbox + 3, mxy);
  }
}
__device__ __forceinline__ uint32_t spread8(uint32_t v) {  // 8 bits -> every other bit of 16
  v &= 0xFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__global__ void k_sort_keys(const double2* __restrict__ xy, const int32_t* __restrict__ tri, int64_t V, int64_t T,
                            const unsigned long long* __restrict__ bbox, uint32_t* __restrict__ key,
                            uint32_t* hist) {
  pdl_enter();
  const double x0 = of_ord(bbox[0]), x1 = of_ord(bbox[1]), y0 = of_ord(bbox[2]), y1 = of_ord(bbox[3]);
  const double sx = x1 > x0 ? 255.999 / (x1 - x0) : 0.0, sy = y1 > y0 ? 255.999 / (y1 - y0) : 0.0;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < T; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = tri[3 * f];
    // (a dangling index is reported by the build; any cell will do)
    const double2 p = (uint64_t)v < (uint64_t)V ? __ldg(xy + v) : make_double2(x0, y0);
    const uint32_t qx = (uint32_t)fmin(fmax((p.x - x0) * sx, 0.0), 255.0);
    const uint32_t qy = (uint32_t)fmin(fmax((p.y - y0) * sy, 0.0), 255.0);
    const uint32_t cell = spread8(qx) | (spread8(qy) << 1);
    key[f] = cell;
    // (neighbouring triangles share cells: one atomic per distinct cell of the warp)
    const uint32_t peers = __match_any_sync(__activemask(), cell);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[cell], (uint32_t)__popc(peers));
  }
}
// exclusive scan of the cell counts in place: one block of 1024 threads, warp w owns the
// 8,192 cells from 8,192 w on, read lane-strided (coalesced), two passes
__global__ void __launch_bounds__(1024) k_sort_scan(uint32_t* hist) {
  pdl_enter();
  constexpr int per = (int)(kSortCells / 32);  // cells per warp
  __shared__ uint32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t* h = hist + (int64_t)wid * per;
  uint32_t sum = 0;
#pragma unroll 8
  for (int i = lane; i < per; i += 32) sum += h[i];
  sum = __reduce_add_sync(0xffffffffu, sum);
  if (lane == 0) wsum[wid] = sum;
  __syncthreads();
  if (wid == 0) {
    const uint32_t w = wsum[lane];
    uint32_t iw = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, iw, o);
      if (lane >= o) iw += a;
    }
    wsum[lane] = iw - w;
  }
  __syncthreads();
  uint32_t carry = wsum[wid];
  for (int i0 = 0; i0 < per; i0 += 32) {
    const uint32_t c = h[i0 + lane];
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    h[i0 + lane] = carry + inc - c;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}
__global__ void k_sort_scatter(int64_t T, const uint32_t* __restrict__ key, uint32_t* cursor, int32_t* __restrict__ perm) {
  pdl_enter();
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < T; f += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t cell = key[f];
    const uint32_t m = __activemask(), peers = __match_any_sync(m, cell);
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&cursor[cell], (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    perm[base + __popc(peers & ((1u << lane) - 1))] = (int32_t)f;
  }
}

Tiling make_tiling(int64_t T, int64_t R, bool sorted) {
  Tiling g;
  if (sorted) {
    g.mode = kTileSorted;
    g.ntiles = (T + kTileTris - 1) / kTileTris;
  } else if (R > 0 && T % R == 0) {
    g.mode = kTileGrid;
    g.R = R;
    g.nrows = T / R;
    g.ntc = (R + kGridTW - 1) / kGridTW;
    g.ntiles = (g.nrows + kGridTH - 1) / kGridTH * g.ntc;
  } else {
    g.ntiles = (T + kTileTris - 1) / kTileTris;
  }
  return g;
}

// Per-device launch setup: the dynamic shared-memory attribute of k_tile belongs to each
// device's context, so it is set once per device id (a relaxed bit-set under a mutex;
// the SM count is cached next to it).
static std::mutex g_dev_mu;
static uint64_t g_dev_ready = 0;  // bit d: device d configured
static int g_dev_sms[64];

static int device_setup(int* n_sm) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (dev >= 64 || !((g_dev_ready >> dev) & 1)) {
    if (cudaFuncSetAttribute(k_tile<kTileContig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem) != cudaSuccess ||
        cudaFuncSetAttribute(k_tile<kTileGrid>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmemGrid) != cudaSuccess ||
        cudaFuncSetAttribute(k_tile<kTileSorted>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmemGrid) != cudaSuccess)
      return -1;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    if (dev >= 64) { *n_sm = sms; return 0; }  // (not cached)
    g_dev_sms[dev] = sms;
    g_dev_ready |= uint64_t(1) << dev;
  }
  *n_sm = g_dev_sms[dev];
  return 0;
}

static int64_t prefetch_distance(int n_sm) {
  // L2 prefetch distance in tiles (default: one per SM, measured best of {0, 148, 296, 444, 592} on config 3);
  // POLYLLA_PREFETCH_DIST overrides it (<= 0 disables the prefetch) for experiments
  static const int64_t pf_env = [] {
    const char* env = std::getenv("POLYLLA_PREFETCH_DIST");
    // INT64_MIN: unset (one tile per SM); <= 0: no prefetch
    return env ? (int64_t)std::atoll(env) : INT64_MIN;
  }();
  return pf_env == INT64_MIN ? (int64_t)n_sm : pf_env <= 0 ? int64_t(1) << 40 : pf_env;
}

// the start of a build: counters zeroed, per-device setup
int launch_build_begin(Ctx* c, cudaStream_t s) {
  if (cudaMemsetAsync(c->ctr, 0, sizeof(DevCounters), s) != cudaSuccess) return -1;
  if (c->tiling.mode != kTileContig) {  // grid / sorted tiles OR their words into the bit-vectors: zero them
    const size_t wb = (size_t)c->n_words * 4;
    if (cudaMemsetAsync(c->F0, 0, (size_t)(c->TB - c->F0) * 4 + wb, s) != cudaSuccess ||
        cudaMemsetAsync(c->C, 0, wb, s) != cudaSuccess || cudaMemsetAsync(c->SDB, 0, wb, s) != cudaSuccess ||
        cudaMemsetAsync(c->wlen, 0, wb, s) != cudaSuccess || cudaMemsetAsync(c->BB, 0, wb, s) != cudaSuccess)
      return -1;
  }
  if (c->tiling.mode == kTileSorted) {  // the triangle order of the sorted tiling
    const unsigned g = 148 * 8;
    launch_k(k_sort_init, g, 256, 0, s, c->sort_bbox, c->sort_hist, kSortCells);
    launch_k(k_sort_bbox, g, 256, 0, s, reinterpret_cast<const double2*>(c->xy), c->V, c->sort_bbox);
    launch_k(k_sort_keys, g, 256, 0, s, reinterpret_cast<const double2*>(c->xy), c->tri, c->V, c->T, c->sort_bbox,
                                  c->sort_key, c->sort_hist);
    launch_k(k_sort_scan, 1, 1024, 0, s, c->sort_hist);
    launch_k(k_sort_scatter, g, 256, 0, s, c->T, c->sort_key, c->sort_hist, const_cast<int32_t*>(c->tiling.perm));
    if (cudaGetLastError() != cudaSuccess) return -1;
  }
  int n_sm = 0;
  return device_setup(&n_sm);
}

// k_tile over tiles [t0, t1)
int launch_build_tiles(Ctx* c, cudaStream_t s, int64_t t0, int64_t t1) {
  if (t1 <= t0) return 0;
  int n_sm = 0;
  if (device_setup(&n_sm) != 0) return -1;
  const int64_t pf_dist = prefetch_distance(n_sm);
  const int64_t bv_stride = c->F1 - c->F0;  // F0, F1, S, TB are equally spaced (capi.cu layout)
  if (c->S - c->F1 != bv_stride || c->TB - c->S != bv_stride) return -1;
  prof_mark(s, "k_tile");
  auto kt = c->tiling.mode == kTileGrid ? k_tile<kTileGrid> : c->tiling.mode == kTileSorted ? k_tile<kTileSorted>
                                                                                         : k_tile<kTileContig>;
  launch_k(kt, (unsigned)(t1 - t0), kTileThreads, c->tiling.mode != kTileContig ? kTileSmemGrid : kTileSmem, s, reinterpret_cast<const double2*>(c->xy), c->tri, c->V, c->T,
                                                          c->origin, c->twin, c->next, c->lcode, c->F0, bv_stride, c->C,
                                                          c->len, c->wlen, c->left_key, c->left_e, c->def_e, c->SDB,
                                                          c->cnt_ld, c->ctr, pf_dist, t0, c->tiling);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int launch_build(Ctx* c, cudaStream_t s) {
  const int64_t tiles = c->tiling.ntiles;
  if (launch_build_begin(c, s) != 0) return -1;
  const int n = launch_build_tiles(c, s, 0, tiles);
  if (n < 0) return -1;
  const int m = launch_build_rest(c, s);
  return m < 0 ? -1 : n + m;
}

// everything after the tiles: leftover match, border half-edges and their chain
int launch_build_rest(Ctx* c, cudaStream_t s) {
  int n = 0;
  const int64_t tiles = c->tiling.ntiles;
  const int grid = 148 * 32;  // enough threads for ~1 leftover each on 10M-vertex meshes (latency-bound)
  prof_mark(s, "k_left_match");
  uint32_t* ehash = static_cast<uint32_t*>(c->ehash);
  launch_k(k_hash_clear, grid, 256, 0, s, c->ctr, ehash, c->hash_cap_max, c->V, c->T);
#ifndef POLYLLA_LEFT_THREADS
#define POLYLLA_LEFT_THREADS 256  // 128 / 256 / 384 / 512 measured: 128-256 best
#endif
  const unsigned seg_grid = (unsigned)(tiles < 148 * 16 ? tiles : 148 * 16);
  const unsigned left_grid = (unsigned)(tiles < 148 * (4096 / POLYLLA_LEFT_THREADS) ? tiles : 148 * (4096 / POLYLLA_LEFT_THREADS));
  launch_k(k_left_insert, left_grid, POLYLLA_LEFT_THREADS, 0, s, c->ctr, tiles, c->T, c->tiling, c->cnt_ld, c->left_key,
                                                           c->left_e, c->twin, ehash);
  if (c->tiling.mode != kTileContig) {  // grid / sorted tiles: the border ranking by bit order
    const int64_t nchunks = (c->n_words + kBBChunk - 1) / kBBChunk;
    launch_k(k_bb_mark, seg_grid, kSegThreads, 0, s, c->ctr, tiles, c->T, c->tiling, c->cnt_ld, c->left_e, c->left_key, c->BB);
    launch_k(k_bb_count, (unsigned)((nchunks + 7) / 8), 256, 0, s, c->ctr, c->n_words, nchunks, c->BB, c->bcnt);
    n += 3;
    prof_mark(s, "k_border_scan");
    launch_k(k_border_scan, 1, kBorderScanThreads, 0, s, c->ctr, nchunks, 3 * c->T, c->Bmax, c->bcnt);
    launch_k(k_bb_emit, (unsigned)((nchunks + 7) / 8), 256, 0, s, c->ctr, c->n_words, nchunks, 3 * c->T, c->BB, c->bcnt,
                                                             c->origin, c->twin, c->vmap);
    n += 2;
  } else {
    hid* blist = reinterpret_cast<hid*>(c->left_key);  // dead after k_left_insert
    launch_k(k_border_rank, seg_grid, kSegThreads, 0, s, c->ctr, tiles, c->cnt_ld, c->left_e, c->left_key, blist, c->bcnt);
    n += 3;
    prof_mark(s, "k_border_scan");
    launch_k(k_border_scan, 1, kBorderScanThreads, 0, s, c->ctr, tiles, 3 * c->T, c->Bmax, c->bcnt);
    launch_k(k_border_emit, seg_grid, kSegThreads, 0, s, c->ctr, tiles, 3 * c->T, blist, c->bcnt, c->origin, c->twin,
                                                   c->vmap);
    n += 2;
  }
  prof_mark(s, "k_border_next");
  launch_k(k_border_next, grid, 256, 0, s, c->ctr, 3 * c->T, c->origin, c->twin, c->vmap, c->next);
  ++n;
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? n : -1;
}

}  // namespace polylla
