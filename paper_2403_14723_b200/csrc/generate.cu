// generate.cu -- repair, seed landing, canonical seeds, compaction
// ("Label extra seed and frontier edges" (Alg. 10), "Search frontier
// edges for each seed edge" (Alg. 12), "Overwrite seeds", "Scan and compact").
//
//   k_repair_mid     one thread per barrier tip (bit-vector TB, set where next == twin):
//                    d = degree(v); m = sweep_out^k(e0), k = floor((d-1)/2) (R5) from the
//                    tip's outgoing frontier half-edge e0; F1[m] = F1[twin m] = 1; both
//                    halves become seeds (bit-vector SDB).  Topology only -> snapshot (R6).
//   k_repair_rewire  one thread per touched vertex w (the tip v and the far end u of m):
//                    recompute next[p] for every incoming frontier half-edge p of w with
//                    the F1 bits (the only next values repair can change).
//   k_seed_walk      one thread per seed of SDB (deferred by k_tile / the fixup, repair
//                    halves; expanded per warp into a shared queue): rotate to the first frontier
//                    half-edge (Alg. 12), walk the polygon through next, keep the minimum
//                    id as the canonical seed and its loop length (Overwrite seeds,
//                    PAPER.md L816).  Duplicate walks of one polygon write the same values.
//   canon scan       per build tile: #canonical seeds, sum of their loop lengths, #F1;
//                    one block scans the tiles (k_emit finishes ranks and offsets inside
//                    each tile); checks sum(len) == #interior F1 half-edges (R12).
#include "internal.cuh"

namespace polylla {

__device__ __forceinline__ bool f1_of(const uint32_t* __restrict__ F1, int64_t T3, hid x) {
  return x >= T3 || bit_of(F1, x);
}

// The tips of the bit-vector TB (set by k_tile and the label fixup), balanced over warps
// (warp_foreach_bit) and compacted (one atomic per round of 32) into tips[] / aff[].
#ifndef POLYLLA_REPAIR_THREADS
#define POLYLLA_REPAIR_THREADS 128
#endif
constexpr int kRepairThreads = POLYLLA_REPAIR_THREADS;
#ifndef POLYLLA_REPAIR_DYN
#define POLYLLA_REPAIR_DYN 1
#endif
#ifndef POLYLLA_SEED_BURST
#define POLYLLA_SEED_BURST 4
#endif
constexpr int kSeedBurst = POLYLLA_SEED_BURST;  // walk steps between per-lane refills (k_repair_mid, k_seed_walk)
#ifndef POLYLLA_ROT_MAX
#define POLYLLA_ROT_MAX 16
#endif
// rotations up to this degree are walked once and kept in shared memory (the rewire; a
// per-thread local array of 32 had 128-B stack frames spilling to L2: 2048 threads x 128 B
// per SM)
constexpr int kRotMax = POLYLLA_ROT_MAX;
__global__ void __launch_bounds__(kRepairThreads)
    k_repair_mid(int64_t T, int64_t n_words, const uint32_t* __restrict__ TB, const hid* __restrict__ twin,
                 uint32_t* F1, uint32_t* SDB, hid* __restrict__ tips, hid* __restrict__ aff, DevCounters* ctr) {
  pdl_enter();
  __shared__ hid queue[kRepairThreads / 32][kBitQueue];
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int lane = threadIdx.x & 31;
#if POLYLLA_REPAIR_DYN
  // per-lane refill (as in k_seed_walk): a lane done with its tip takes the queue's next one;
  // the degree walk and the middle-edge walk are the same step (x <- next_in(twin x))
  warp_foreach_bit<true>(TB, n_words, queue[threadIdx.x >> 5], [&](const hid* q, int fill) {
    int base = 0;
    if (lane == 0) base = atomicAdd(&ctr->n_tips, fill);
    base = __shfl_sync(0xffffffffu, base, 0);
    int head = 0, idx = 0;
    bool active = false, second = false;
    hid e0 = 0, x = 0;
    int64_t d = 0, st = 0, target = 0;
    while (true) {
      const uint32_t idle = __ballot_sync(0xffffffffu, !active);
      if (head < fill && idle) {
        const int my = head + __popc(idle & ((1u << lane) - 1));
        head += __popc(idle);
        if (!active && my < fill) {
          const hid e = q[my];
          idx = base + my;
          tips[idx] = e;
          e0 = twin[e];  // the tip's only outgoing frontier half-edge
          x = e0;
          d = 0;
          second = false;
          active = true;
        }
      }
      if (!__any_sync(0xffffffffu, active)) {
        if (head >= fill) break;
        continue;
      }
#pragma unroll 1
      for (int k = 0; k < kSeedBurst && active; ++k) {
        bool done = false;
        if (!second) {  // degree(v): rotation closure about v (an interior vertex); deg(v) <= 3T
          const hid tx = twin[x];
          if (tx >= T3 || ++d > T3) {
            raise_status(ctr, ST_WALK);
            aff[2 * idx] = aff[2 * idx + 1] = e0;
            active = false;
            break;
          }
          x = next_in(tx);
          if (x == e0) {  // floor((d-1)/2) CWvertexEdge steps (R1, R5) from e0
            second = true;
            target = (d - 1) / 2;
            st = 0;
            done = target == 0;
          }
        } else {
          x = next_in(twin[x]);
          done = ++st == target;
        }
        if (done) {
          const hid m = x, tm = twin[m];
          atomicOr(&F1[m >> 5], 1u << (m & 31));
          atomicOr(&F1[tm >> 5], 1u << (tm & 31));
          atomicOr(&SDB[m >> 5], 1u << (m & 31));  // both halves seed the split polygons
          atomicOr(&SDB[tm >> 5], 1u << (tm & 31));
          aff[2 * idx] = e0;      // outgoing from v
          aff[2 * idx + 1] = tm;  // outgoing from u = target(m)
          active = false;
        }
      }
    }
  });
#else
  warp_foreach_bit(TB, n_words, queue[threadIdx.x >> 5], [&](hid e, bool valid) {
    const uint32_t m32 = __ballot_sync(0xffffffffu, valid);
    int base = 0;
    if (lane == 0) base = atomicAdd(&ctr->n_tips, __popc(m32));
    const int i = __shfl_sync(0xffffffffu, base, 0) + __popc(m32 & ((1u << lane) - 1));
    if (!valid) return;
    const hid e0 = twin[e];  // the tip's only outgoing frontier half-edge
    hid x = e0;
    int64_t d = 0;
    bool ok = true;
    do {  // degree(v): rotation closure about v (an interior vertex); deg(v) <= 3T
      const hid tx = twin[x];
      if (tx >= T3 || ++d > T3) { ok = false; break; }
      x = next_in(tx);
    } while (x != e0);
    tips[i] = e;
    if (!ok) {
      raise_status(ctr, ST_WALK);
      aff[2 * i] = aff[2 * i + 1] = e0;
      return;
    }
    hid m = e0;  // floor((d-1)/2) CWvertexEdge steps (R1, R5), again along the walked rotation (L1 hits)
    for (int64_t k = 0; k < (d - 1) / 2; ++k) m = next_in(twin[m]);
    const hid tm = twin[m];
    atomicOr(&F1[m >> 5], 1u << (m & 31));
    atomicOr(&F1[tm >> 5], 1u << (tm & 31));
    atomicOr(&SDB[m >> 5], 1u << (m & 31));  // both halves seed the split polygons
    atomicOr(&SDB[tm >> 5], 1u << (tm & 31));
    aff[2 * i] = e0;     // outgoing from v
    aff[2 * i + 1] = tm; // outgoing from u = target(m)
  });
#endif
}

__global__ void __launch_bounds__(kRepairThreads)
    k_repair_rewire(int64_t T, const hid* __restrict__ twin, const uint32_t* __restrict__ F1,
                    const hid* __restrict__ aff, hid* next, DevCounters* ctr) {
  pdl_enter();
  __shared__ hid rot_s[kRotMax][kRepairThreads];  // (entry k of this thread's rotation: rot_s[k][tid])
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int64_t H = T3 + ctr->n_border;  // walk bound (a rotation about w has <= deg(w) <= H steps)
  const int32_t n = 2 * ctr->n_tips;
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const hid o = aff[j];
    // one walk around w collects its outgoing half-edges in sweep order (R1; the border
    // chain at the hull); the next F1 half-edge after each incoming p = prev_in(y_i) is
    // then the first frontier y_m, m >= i cyclically -- what a rotation from y_i finds
    hid* const rot = &rot_s[0][threadIdx.x];  // rot[i * kRepairThreads]
    int d = 0;
    bool fits = true, ok = true;
    {
      hid y = o;
      int64_t guard = 0;
      do {
        if (d < kRotMax) rot[d * kRepairThreads] = y; else fits = false;
        ++d;
        const hid ty = twin[y];
        y = ty >= T3 ? next[ty] : next_in(ty);
        if (++guard > H) { ok = false; break; }
      } while (y != o);
    }
    if (!ok) { raise_status(ctr, ST_WALK); return; }
    if (fits) {
      uint32_t fo = 0, fi = 0;  // bit i: y_i frontier (F1 or border) / p_i = prev_in(y_i) an interior F1 half-edge
      for (int i = 0; i < d; ++i) {
        const hid y = rot[i * kRepairThreads];
        fo |= (uint32_t)f1_of(F1, T3, y) << i;
        if (y < T3) fi |= (uint32_t)f1_of(F1, T3, prev_in(y)) << i;
      }
      if (fi && !fo) { raise_status(ctr, ST_WALK); return; }  // (a rotation without a frontier half-edge)
      for (uint32_t b = fi; b; b &= b - 1) {
        const int i = __ffs(b) - 1;
        const uint32_t ahead = fo >> i;  // (i < 32)
        const int m = ahead ? i + __ffs(ahead) - 1 : __ffs(fo) - 1;
        next[prev_in(rot[i * kRepairThreads])] = rot[m * kRepairThreads];
      }
      continue;
    }
    // (degree above kRotMax: the rotation walked per incoming F1 half-edge)
    hid y = o;
    int64_t guard = 0;
    do {
      if (y < T3) {
        const hid p = prev_in(y);  // incoming to w in y's triangle; next_in(p) = y
        if (f1_of(F1, T3, p)) {
          hid x = y;
          int64_t steps = 0;
          while (!f1_of(F1, T3, x) && ++steps <= H) x = next_in(twin[x]);
          if (steps > H) {  // the rotation to the next F1 half-edge did not close
            raise_status(ctr, ST_WALK);
            return;
          }
          next[p] = x;
        }
      }
      const hid ty = twin[y];
      y = ty >= T3 ? next[ty] : next_in(ty);  // full rotation about w (border chain at the hull)
      if (++guard > H) { raise_status(ctr, ST_WALK); break; }
    } while (y != o);
  }
}

#ifndef POLYLLA_SEED_THREADS
#define POLYLLA_SEED_THREADS 256
#endif
constexpr int kSeedThreads = POLYLLA_SEED_THREADS;
#ifndef POLYLLA_SEED_DYN
#define POLYLLA_SEED_DYN 1
#endif


__device__ __forceinline__ void process_seed(hid s, int64_t T3, int64_t H, const hid* __restrict__ twin,
                                             const hid* __restrict__ next, const uint32_t* __restrict__ F1,
                                             uint32_t* C, uint8_t* len, int32_t* wlen, DevCounters* ctr) {
  hid x = s;
  int64_t steps = 0;
  while (!f1_of(F1, T3, x)) {  // Alg. 12: rotate (sweep_out) to a frontier half-edge (<= deg <= 3T steps)
    x = next_in(twin[x]);
    if (++steps > T3 || x == s) { raise_status(ctr, ST_WALK); return; }
  }
  hid mn = x, y = x;
  int64_t n = 0;
  do {  // Overwrite seeds: walk the polygon, keep the minimum index
    mn = min(mn, y);
    y = next[y];
    if (++n > H) { raise_status(ctr, ST_WALK); return; }
  } while (y != x);
  len[mn] = len_code(n);
  const uint32_t bit = 1u << (mn & 31);
  if (!(atomicOr(&C[mn >> 5], bit) & bit)) atomicAdd(&wlen[mn >> 5], (int32_t)n);  // first setter only
}

// The seeds of the bit-vector SDB: those k_tile could not close inside their tile, those
// the label fixup found, and both halves of every middle edge of the repair; balanced
// over warps (warp_foreach_bit), one seed per lane.
__global__ void __launch_bounds__(kSeedThreads)
    k_seed_walk(int64_t T, int64_t n_words, const uint32_t* __restrict__ SDB, const hid* __restrict__ twin,
                const hid* __restrict__ next, const uint32_t* __restrict__ F1, uint32_t* C, uint8_t* len,
                int32_t* wlen, DevCounters* ctr) {
  pdl_enter();
  __shared__ hid queue[kSeedThreads / 32][kBitQueue];
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int64_t H = T3 + ctr->n_border;
#if POLYLLA_SEED_DYN
  // a lane that closes its loop takes the next seed of the warp's queue (ballot of the idle
  // lanes, ranks by popcount) instead of waiting for the round's longest walk; walks
  // advance kSeedBurst steps between refills
  const int lane = threadIdx.x & 31;
  const int n = warp_foreach_bit<true>(SDB, n_words, queue[threadIdx.x >> 5], [&](const hid* q, int fill) {
    int head = 0;
    bool active = false;
    hid x = 0, y = 0, mn = 0;
    int64_t cnt = 0;
    while (true) {
      const uint32_t idle = __ballot_sync(0xffffffffu, !active);
      if (head < fill && idle) {
        const int my = head + __popc(idle & ((1u << lane) - 1));
        head += __popc(idle);
        if (!active && my < fill) {
          const hid s = q[my];
          hid xx = s;
          int64_t steps = 0;
          bool ok = true;
          while (!f1_of(F1, T3, xx)) {  // Alg. 12: rotate (sweep_out) to a frontier half-edge
            xx = next_in(twin[xx]);
            if (++steps > T3 || xx == s) { raise_status(ctr, ST_WALK); ok = false; break; }
          }
          if (ok) { active = true; x = y = mn = xx; cnt = 0; }
        }
      }
      if (!__any_sync(0xffffffffu, active)) {
        if (head >= fill) break;
        continue;
      }
#pragma unroll 1
      for (int k = 0; k < kSeedBurst && active; ++k) {  // Overwrite seeds: walk the polygon, keep the minimum
        mn = min(mn, y);
        y = next[y];
        if (++cnt > H) { raise_status(ctr, ST_WALK); active = false; break; }
        if (y == x) {
          len[mn] = len_code(cnt);
          const uint32_t bit = 1u << (mn & 31);
          if (!(atomicOr(&C[mn >> 5], bit) & bit)) atomicAdd(&wlen[mn >> 5], (int32_t)cnt);  // first setter only
          active = false;
        }
      }
    }
  });
#else
  const int n = warp_foreach_bit(SDB, n_words, queue[threadIdx.x >> 5], [&](hid s, bool valid) {
    if (valid) process_seed(s, T3, H, twin, next, F1, C, len, wlen, ctr);
  });
#endif
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(&ctr->n_sdef, (uint32_t)n);
}

// "Scan and compact" at tile granularity: per build tile (192 words
// of 32 half-edges) the number of canonical seeds, the sum of their loop lengths and
// the number of interior F1 half-edges; then one block scans the tiles.  The
// per-polygon ranks and offsets are finished inside the tile by k_emit (extract.cu).
constexpr int kTileWordsG = 3 * kBuildTileTris / 32;  // 192

__global__ void k_canon_tiles(int64_t n_words, int64_t ntiles, const uint32_t* __restrict__ C,
                              const int32_t* __restrict__ wlen, const uint32_t* __restrict__ F1, int32_t* __restrict__ ts,
                              DevCounters* ctr) {
  pdl_enter();
  if (ctr->status) return;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < ntiles; tile += nwarps) {
    int p = 0, l = 0, f = 0;
    for (int k = lane; k < kTileWordsG; k += 32) {
      const int64_t w = tile * kTileWordsG + k;
      if (w < n_words) {
        p += __popc(C[w]);
        l += wlen[w];
        f += __popc(F1[w]);
      }
    }
    p = __reduce_add_sync(0xffffffffu, p);
    l = __reduce_add_sync(0xffffffffu, l);
    f = __reduce_add_sync(0xffffffffu, f);
    if (lane == 0) {
      ts[3 * tile] = p;
      ts[3 * tile + 1] = l;
      ts[3 * tile + 2] = f;
    }
  }
}

// one block of kTopThreads: warp w owns a contiguous run of tiles, read 32 at a time
// (coalesced); pass 1 sums each warp's run, the warp totals are scanned, pass 2 rescans
// the run with its carry and writes the exclusive prefixes of (polygons, loop entries)
// per tile -> tb[2 * tile + {0, 1}]; totals -> P, L; the R12 check sum(len) == #F1
constexpr int kTopThreads = 1024;
__global__ void __launch_bounds__(kTopThreads)
    k_tiles_scan(int64_t ntiles, const int32_t* __restrict__ ts, uint32_t* __restrict__ tb, uint32_t* __restrict__ offsets,
                 DevCounters* ctr) {
  pdl_enter();
  constexpr int NW = kTopThreads / 32;
  __shared__ long long wsum[3][NW];
  if (ctr->status) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t per = ((ntiles + NW - 1) / NW + 31) & ~int64_t(31);
  const int64_t t0 = wid * per, t1 = t0 + per < ntiles ? t0 + per : ntiles;
  long long p = 0, l = 0, f = 0;
  for (int64_t t = t0 + lane; t < t1; t += 32) { p += ts[3 * t]; l += ts[3 * t + 1]; f += ts[3 * t + 2]; }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    p += __shfl_xor_sync(0xffffffffu, p, o);
    l += __shfl_xor_sync(0xffffffffu, l, o);
    f += __shfl_xor_sync(0xffffffffu, f, o);
  }
  if (lane == 0) { wsum[0][wid] = p; wsum[1][wid] = l; wsum[2][wid] = f; }
  __syncthreads();
  if (wid == 0) {
    long long a = wsum[0][lane], b = wsum[1][lane], c = wsum[2][lane];
    long long ia = a, ib = b, ic = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(0xffffffffu, ia, o), y = __shfl_up_sync(0xffffffffu, ib, o),
                      z = __shfl_up_sync(0xffffffffu, ic, o);
      if (lane >= o) { ia += x; ib += y; ic += z; }
    }
    wsum[0][lane] = ia - a;
    wsum[1][lane] = ib - b;
    if (lane == 31) {
      ctr->P = (int32_t)ia;
      ctr->L = (uint32_t)ib;
      ctr->n_f1 = (uint32_t)ic;
      if (ib != ic) raise_status(ctr, ST_UNSEEDED);  // R12: a frontier loop without a seed
      offsets[ia] = (uint32_t)ib;
    }
  }
  __syncthreads();
  long long cp = wsum[0][wid], cl = wsum[1][wid];
  for (int64_t tb0 = t0; tb0 < t1; tb0 += 32) {
    const int64_t t = tb0 + lane;
    const int vp = t < t1 ? ts[3 * t] : 0, vl = t < t1 ? ts[3 * t + 1] : 0;
    int ip = vp, il = vl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, ip, o), y = __shfl_up_sync(0xffffffffu, il, o);
      if (lane >= o) { ip += x; il += y; }
    }
    if (t < t1) {
      tb[2 * t] = (uint32_t)(cp + ip - vp);
      tb[2 * t + 1] = (uint32_t)(cl + il - vl);
    }
    cp += __shfl_sync(0xffffffffu, ip, 31);
    cl += __shfl_sync(0xffffffffu, il, 31);
  }
}

int launch_canon_scan(Ctx* c, cudaStream_t s);

int launch_generate(Ctx* c, cudaStream_t s) {
  int n = 0;
  if (c->next_pre) cudaMemcpyAsync(c->next_pre, c->next, (size_t)c->Hmax * 4, cudaMemcpyDeviceToDevice, s);
  prof_mark(s, "k_repair");
  launch_k(k_repair_mid, 148 * (1536 / kRepairThreads), kRepairThreads, 0, s, c->T, c->n_words, c->TB, c->twin, c->F1, c->SDB, c->tips, c->aff, c->ctr);
  launch_k(k_repair_rewire, 148 * (4096 / kRepairThreads), kRepairThreads, 0, s, c->T, c->twin, c->F1, c->aff, c->next, c->ctr);
  prof_mark(s, "k_seed_walk");
  // (the canonical bit-vector C was written in full by k_tile; global walks OR into it)
  launch_k(k_seed_walk, 148 * (2048 / kSeedThreads), kSeedThreads, 0, s, c->T, c->n_words, c->SDB, c->twin, c->next, c->F1, c->C, c->len,
                                               c->wlen, c->ctr);
  n += 3;
  const int m = launch_canon_scan(c, s);
  if (m < 0) return -1;
  n += m;
  return cudaGetLastError() == cudaSuccess ? n : -1;
}

int launch_canon_scan(Ctx* c, cudaStream_t s) {
  prof_mark(s, "k_canon_scan");
  const int64_t tiles = (c->T + kBuildTileTris - 1) / kBuildTileTris;
  launch_k(k_canon_tiles, (unsigned)((tiles + 7) / 8), 256, 0, s, c->n_words, tiles, c->C, c->wlen, c->F1, c->tsum, c->ctr);
  launch_k(k_tiles_scan, 1, kTopThreads, 0, s, tiles, c->tsum, c->tbase, c->offsets, c->ctr);
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace polylla
