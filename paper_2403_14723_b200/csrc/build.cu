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
//     - half-edges whose twin is outside the tile are appended to a leftover list.
//   k_left_insert / k_left_unmatched  -- global hash over the leftovers only;
//   border scan (scan.cuh)             -- border ids 3T + rank(e) (R9), twin/origin of
//                                         border half-edges, border-vertex hash;
//   k_border_next                      -- next(b) = border half-edge leaving target(b).
#include "internal.cuh"
#include "scan.cuh"

namespace polylla {

constexpr int kTileTris = 2048;
constexpr int kTileHE = 3 * kTileTris;   // 6144 half-edges = 192 bit-vector words
constexpr int kTileSlots = 8192;         // pow2 hash slots, >= 2.4x the unique keys of a tile
constexpr int kTileThreads = 512;
constexpr int kTileWalk = 64;            // longer in-tile rotations are deferred to the fixup
// shared memory: tri_s int32[kTileHE] | tw_s int16[kTileHE] | slot uint16[kTileSlots] | lc_s u8[kTileTris]
constexpr size_t kTileSmem = kTileHE * 4 + kTileHE * 2 + kTileSlots * 2 + kTileTris;  // 55,296 B -> 3-4 CTAs/SM
constexpr uint16_t kEmpty16 = 0xFFFFu, kPaired16 = 0x8000u;

__device__ __forceinline__ int32_t next_local(int32_t j) { return (j % 3 == 2) ? j - 2 : j + 1; }

__device__ __forceinline__ double sq_len(double2 p, double2 q) {
  // |q - p|^2 = dx*dx + dy*dy, dx = x[target] - x[origin]; IEEE RN, no FMA (R11)
  const double dx = __dsub_rn(q.x, p.x), dy = __dsub_rn(q.y, p.y);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// L2 policies: keep the randomly gathered coordinates (vertex ids are spatially random)
// resident, stream the triangle tile through.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_xy(const double2* ptr, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(ptr), "l"(pol));
  return r;
}

// One CTA per tile of kTileTris triangles.  Phases (PAPER.md section in brackets):
//  P0 stage the triangle tile (coalesced, streaming)
//  P1 per triangle: checks, CCW orientation (R10), longest edge Lcode (Alg. 2/7)
//  P2 tile-local twin matching in a shared-memory hash on (min, max)      [Sec. 4]
//  P3 write origin/twin (coalesced); cross-tile half-edges -> leftover list
//  P4 per half-edge whose twin is in the tile: frontier/seed bits (Alg. 8-9) and the
//     unlink rewire (Alg. 11) with the rotation walk in shared memory; tips (next ==
//     twin).  Half-edges that need a twin outside the tile are deferred to
//     k_label_fixup (label phase), which sees the completed global twin array.
__global__ void __launch_bounds__(kTileThreads, 3)
    k_tile(const double2* __restrict__ xy, const int32_t* __restrict__ tri, int64_t V, int64_t T,
           int32_t* __restrict__ origin, int32_t* __restrict__ twin, int32_t* __restrict__ next,
           uint8_t* __restrict__ lcode, uint32_t* __restrict__ F0, uint32_t* __restrict__ F1,
           uint32_t* __restrict__ S, unsigned long long* __restrict__ left_key, int32_t* __restrict__ left_e,
           int32_t* __restrict__ def_e, int32_t* __restrict__ tips, DevCounters* ctr) {
  extern __shared__ __align__(16) unsigned char smem_tile[];
  int32_t* tri_s = reinterpret_cast<int32_t*>(smem_tile);
  int16_t* tw_s = reinterpret_cast<int16_t*>(smem_tile + kTileHE * 4);
  uint16_t* slot = reinterpret_cast<uint16_t*>(smem_tile + kTileHE * 6);
  uint8_t* lc_s = smem_tile + kTileHE * 6 + kTileSlots * 2;

  const int64_t f0 = (int64_t)blockIdx.x * kTileTris;
  const int nt = (int)(T - f0 < kTileTris ? T - f0 : kTileTris);
  const int nhe = 3 * nt;
  const int64_t e0 = 3 * f0;
  const int tid = threadIdx.x, lane = tid & 31;

  // ---- P0
  const int32_t* src = tri + e0;
  if (nhe == kTileHE && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    const int4* s4 = reinterpret_cast<const int4*>(src);
    for (int i = tid; i < kTileHE / 4; i += kTileThreads) reinterpret_cast<int4*>(tri_s)[i] = __ldcs(s4 + i);
  } else {
    for (int i = tid; i < nhe; i += kTileThreads) tri_s[i] = __ldcs(src + i);
  }
  for (int i = tid; i < kTileSlots / 2; i += kTileThreads) reinterpret_cast<uint32_t*>(slot)[i] = 0xFFFFFFFFu;
  for (int i = tid; i < kTileHE / 2; i += kTileThreads) reinterpret_cast<uint32_t*>(tw_s)[i] = 0xFFFFFFFFu;
  __syncthreads();

  // ---- P1
  const uint64_t pol = policy_evict_last();
  uint32_t bad = 0;
  int flips = 0;
#pragma unroll 4
  for (int t = tid; t < nt; t += kTileThreads) {
    int32_t a = tri_s[3 * t], b = tri_s[3 * t + 1], c = tri_s[3 * t + 2];
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
    lcode[f0 + t] = (uint8_t)k;
    tri_s[3 * t] = a; tri_s[3 * t + 1] = b; tri_s[3 * t + 2] = c;
  }
  flips = __reduce_add_sync(0xffffffffu, flips);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0) {
    if (flips) atomicAdd(&ctr->n_flips, flips);
    if (bad) raise_status(ctr, bad);
  }
  __syncthreads();

  // ---- P2
  uint32_t nm = 0;
  for (int j = tid; j < nhe; j += kTileThreads) {
    const int32_t o = tri_s[j], tg = tri_s[next_local(j)];
    const uint32_t lo = (uint32_t)min(o, tg), hi = (uint32_t)max(o, tg);
    uint32_t h = mix32(lo, hi) & (kTileSlots - 1);
    for (int probe = 0; probe < kTileSlots; ++probe) {
      uint16_t s = slot[h];
      if (s == kEmpty16) {
        const uint16_t old = atomicCAS(&slot[h], kEmpty16, (uint16_t)j);
        if (old == kEmpty16) break;  // first of its key
        s = old;
      }
      const int32_t sj = s & ~kPaired16;
      const int32_t so = tri_s[sj], st = tri_s[next_local(sj)];
      if ((uint32_t)min(so, st) == lo && (uint32_t)max(so, st) == hi) {
        if ((s & kPaired16) || so == o) { nm = ST_NONMANIFOLD_EDGE; break; }
        if (atomicCAS(&slot[h], s, (uint16_t)(s | kPaired16)) != s) { nm = ST_NONMANIFOLD_EDGE; break; }
        tw_s[j] = (int16_t)sj;
        tw_s[sj] = (int16_t)j;
        break;
      }
      h = (h + 1) & (kTileSlots - 1);
    }
  }
  if (nm) raise_status(ctr, nm);
  __syncthreads();

  // ---- P3 + P4 (one pass over the tile's half-edges, warp-aligned for the ballots)
  for (int base = 0; base < nhe; base += kTileThreads) {
    const int j = base + tid;
    const bool valid = j < nhe;
    bool fr = false, sd = false, tip = false, deferred = false, left = false;
    if (valid) {
      const int32_t t = tw_s[j];
      __stcs(origin + e0 + j, tri_s[j]);
      __stcs(twin + e0 + j, t >= 0 ? (int32_t)(e0 + t) : -1);
      if (t < 0) {
        left = true;
        deferred = true;
      } else {
        const bool Le = lc_s[j / 3] == j % 3;
        const bool Lt = lc_s[t / 3] == t % 3;
        fr = !Le && !Lt;
        sd = Le && Lt && j < t;
        int32_t nx = next_local(j);
        if (fr) {
          int32_t x = nx;
          for (int steps = 0;; ++steps) {
            const int32_t tx = tw_s[x];
            if (tx < 0 || steps >= kTileWalk) { deferred = true; break; }
            if (lc_s[x / 3] != x % 3 && lc_s[tx / 3] != tx % 3) break;  // frontier edge
            x = next_local(tx);                                        // cross it (sweep_out)
          }
          nx = x;
          tip = !deferred && x == t;
        }
        if (!deferred) __stcs(next + e0 + j, (int32_t)(e0 + nx));
        else fr = sd = false;  // the fixup sets every bit of a deferred half-edge
      }
    }
    const uint32_t fw = __ballot_sync(0xffffffffu, fr);
    const uint32_t sw = __ballot_sync(0xffffffffu, sd);
    const uint32_t tm = __ballot_sync(0xffffffffu, tip);
    const uint32_t dm = __ballot_sync(0xffffffffu, deferred);
    const uint32_t lm = __ballot_sync(0xffffffffu, left);
    const int wbase = j - lane;
    if (lane == 0 && wbase < nhe) {
      const int64_t w = (e0 + wbase) >> 5;
      F0[w] = fw;
      F1[w] = fw;
      S[w] = sw;
    }
    if (lm) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(&ctr->n_left, __popc(lm));
      pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(lm & ((1u << lane) - 1));
      if (left) {
        const int32_t o = tri_s[j], tg = tri_s[next_local(j)];
        const uint64_t lo = (uint32_t)min(o, tg), hi = (uint32_t)max(o, tg);
        left_key[pos] = (lo << 32) | hi;
        left_e[pos] = (int32_t)(e0 + j);
      }
    }
    if (dm) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(&ctr->n_def, __popc(dm));
      pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(dm & ((1u << lane) - 1));
      if (deferred) def_e[pos] = (int32_t)(e0 + j);
    }
    if (tm) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(&ctr->n_tips, __popc(tm));
      pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(tm & ((1u << lane) - 1));
      if (tip) tips[pos] = (int32_t)(e0 + j);
    }
  }
}

__device__ __forceinline__ uint64_t hash_cap_for(int32_t n) {
  uint64_t c = 1024;
  while (c < 2ull * (uint64_t)n) c <<= 1;
  return c;
}

__global__ void k_hash_clear(DevCounters* ctr, uint32_t* ehash, uint32_t* vkey, int64_t cap_max) {
  const uint64_t cap = hash_cap_for(ctr->n_left);
  if ((int64_t)cap > cap_max) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_status(ctr, ST_INTERNAL);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->hash_cap = (uint32_t)cap;
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
    ehash[i] = kEmpty;
    vkey[i] = kEmpty;
  }
}

// global hash over leftover half-edges: pair the two halves of each cross-tile edge
__global__ void k_left_insert(DevCounters* ctr, const unsigned long long* __restrict__ left_key,
                              const int32_t* __restrict__ left_e, const int32_t* __restrict__ origin,
                              int32_t* twin, uint32_t* ehash) {
  if (ctr->status) return;
  const int32_t n = ctr->n_left;
  const uint32_t mask = (uint32_t)ctr->hash_cap - 1;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long key = left_key[i];
    uint32_t h = mix32((uint32_t)(key >> 32), (uint32_t)key) & mask;
    for (uint32_t probe = 0; probe <= mask; ++probe) {
      uint32_t s = ehash[h];
      if (s == kEmpty) {
        const uint32_t old = atomicCAS(&ehash[h], kEmpty, (uint32_t)i);
        if (old == kEmpty) break;
        s = old;
      }
      const int32_t si = (int32_t)(s & ~kPaired);
      if (left_key[si] == key) {
        const int32_t ei = left_e[i], es = left_e[si];
        if ((s & kPaired) || origin[ei] == origin[es] ||
            atomicCAS(&ehash[h], s, s | kPaired) != s) {
          raise_status(ctr, ST_NONMANIFOLD_EDGE);
          break;
        }
        twin[ei] = es;
        twin[es] = ei;
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// mark leftovers that found no partner: they lie on the domain boundary
__global__ void k_left_unmatched(DevCounters* ctr, const int32_t* __restrict__ left_e,
                                 const int32_t* __restrict__ twin, uint32_t* Bd) {
  if (ctr->status) return;
  const int32_t n = ctr->n_left;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t e = left_e[i];
    if (twin[e] < 0) atomicOr(&Bd[e >> 5], 1u << (e & 31));
  }
}

// border records: b = 3T + rank(e) over unmatched interior e (R9)
struct BorderOp {
  const uint32_t* Bd;
  int32_t *origin, *twin;
  uint32_t* vkey;
  int32_t* vval;
  DevCounters* ctr;
  int64_t T3;
  __device__ bool skip() const { return ctr->status != 0; }
  __device__ uint32_t word(int64_t w) const { return Bd[w]; }
  __device__ long long aux(int32_t) const { return 0; }
  __device__ long long extra(int64_t) const { return 0; }
  __device__ void finish(long long cnt, long long, long long) const {
    if (T3 + cnt > 0x7fffffffLL) raise_status(ctr, ST_OVERFLOW);
    ctr->n_border = (int32_t)cnt;
  }
  __device__ void emit(int32_t e, long long rank, long long) const {
    const int32_t b = (int32_t)(T3 + rank);
    const int32_t v = origin[next_in(e)];  // origin(b) = target(e)
    twin[e] = b;
    twin[b] = e;
    origin[b] = v;
    const uint32_t mask = (uint32_t)ctr->hash_cap - 1;
    uint32_t h = mix32((uint32_t)v, 0x5bd1e995u) & mask;
    for (uint32_t probe = 0; probe <= mask; ++probe) {
      const uint32_t old = atomicCAS(&vkey[h], kEmpty, (uint32_t)v);
      if (old == kEmpty) { vval[h] = b; return; }
      if (old == (uint32_t)v) { raise_status(ctr, ST_NONMANIFOLD_VERTEX); return; }
      h = (h + 1) & mask;
    }
    raise_status(ctr, ST_INTERNAL);
  }
};

// next(b) = the border half-edge whose origin is target(b) = origin(twin(b))
__global__ void k_border_next(DevCounters* ctr, int64_t T3, const int32_t* __restrict__ origin,
                              const int32_t* __restrict__ twin, const uint32_t* __restrict__ vkey,
                              const int32_t* __restrict__ vval, int32_t* next) {
  if (ctr->status) return;
  const int32_t nb = ctr->n_border;
  const uint32_t mask = (uint32_t)ctr->hash_cap - 1;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const int32_t b = (int32_t)(T3 + i);
    const uint32_t v = (uint32_t)origin[twin[b]];
    uint32_t h = mix32(v, 0x5bd1e995u) & mask;
    int32_t nx = -1;
    for (uint32_t probe = 0; probe <= mask; ++probe) {
      const uint32_t k = vkey[h];
      if (k == v) { nx = vval[h]; break; }
      if (k == kEmpty) break;
      h = (h + 1) & mask;
    }
    if (nx < 0) raise_status(ctr, ST_NONMANIFOLD_VERTEX);
    next[b] = nx;
  }
}

int launch_build(Ctx* c, cudaStream_t s) {
  int n = 0;
  const int64_t tiles = (c->T + kTileTris - 1) / kTileTris;
  cudaMemsetAsync(c->ctr, 0, sizeof(DevCounters), s);
  cudaMemsetAsync(c->Bd, 0, (size_t)c->n_words * 4, s);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem);
    attr = true;
  }
  prof_mark(s, "k_tile");
  k_tile<<<(unsigned)tiles, kTileThreads, kTileSmem, s>>>(reinterpret_cast<const double2*>(c->xy), c->tri, c->V, c->T,
                                                          c->origin, c->twin, c->next, c->lcode, c->F0, c->F1, c->S,
                                                          c->left_key, c->left_e, c->def_e, c->tips, c->ctr);
  ++n;
  const int grid = 148 * 8;
  prof_mark(s, "k_left_match");
  k_hash_clear<<<grid, 256, 0, s>>>(c->ctr, c->ehash, c->vkey, c->hash_cap_max);
  k_left_insert<<<grid, 256, 0, s>>>(c->ctr, c->left_key, c->left_e, c->origin, c->twin, c->ehash);
  k_left_unmatched<<<grid, 256, 0, s>>>(c->ctr, c->left_e, c->twin, c->Bd);
  n += 3;
  prof_mark(s, "k_border_scan");
  BorderOp op{c->Bd, c->origin, c->twin, c->vkey, c->vval, c->ctr, 3 * c->T};
  const int r = launch_scan(op, c->n_words, c->scan_a, c->scan_b, c->scan_c, s);
  if (r < 0) return -1;
  n += r;
  prof_mark(s, "k_border_next");
  k_border_next<<<grid, 256, 0, s>>>(c->ctr, 3 * c->T, c->origin, c->twin, c->vkey, c->vval, c->next);
  ++n;
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? n : -1;
}

}  // namespace polylla
