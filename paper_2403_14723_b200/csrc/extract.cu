// extract.cu -- polygon extraction ("the seed list is used to rebuild
// each polygon of the output mesh using the next ... queries"), moved on-device and
// fused with the last step of "Scan and compact":
//   seeds[p] = p-th canonical seed, offsets[p] = sum of the earlier loop lengths,
//   loops[offsets[p] + i] = origin[x_i], x_0 = seeds[p], x_{i+1} = next[x_i]   (CSR)
// plus the optional prev array: the inverse of next on frontier and border
// half-edges (their next is a permutation of them), prev_in on the others.
#include "internal.cuh"

namespace polylla {

// One CTA per build tile (kBuildTileTris triangles = 192 words of 32 half-edges):
// warp 0 ranks the words' canonical seeds (C bits) on top of the tile base of
// k_tiles_scan; the seeds are expanded in rank order into a shared queue with their
// loop lengths (len), a block scan turns the lengths into offsets, and each thread then
// walks one polygon: offsets/seeds at the polygon's rank, the loop's vertex ids from
// its canonical seed (the tile's next/origin lines stay in L1 across the CTA's walks).
// Polygons come out in ascending canonical-seed order.
constexpr int kEmitTileWords = 3 * kBuildTileTris / 32;  // 192
// each build tile is emitted by kEmitSub CTAs, one per run of kEmitWords words: a CTA
// holds its shared memory and registers until its longest loop walk ends, so smaller
// parts free them sooner (a part's bases: the tile's, plus the popcounts / per-word length
// sums of the tile's earlier words)
#ifndef POLYLLA_EMIT_SUB
#define POLYLLA_EMIT_SUB 3  // (parts per tile: 1 / 2 / 3 / 6 measured on configs 3 and 5; 3 best, 6 equal)
#endif
constexpr int kEmitSub = POLYLLA_EMIT_SUB;
constexpr int kEmitWords = kEmitTileWords / kEmitSub;
static_assert(kEmitTileWords % kEmitSub == 0 && kEmitWords % 32 == 0, "emission parts of whole lanes of words");
#ifndef POLYLLA_EMIT_THREADS
#define POLYLLA_EMIT_THREADS (384 / POLYLLA_EMIT_SUB)  // (one part per tile: 256/384/512 measured, 384 best; two: 192 / 256)
#endif
constexpr int kEmitThreads = POLYLLA_EMIT_THREADS;
#ifndef POLYLLA_EMIT_Q
#define POLYLLA_EMIT_Q (2048 / POLYLLA_EMIT_SUB)  // (a test variant sets it tiny to force the dense-tile branch)
#endif
constexpr int kEmitQ = POLYLLA_EMIT_Q;  // queue capacity (polygons per tile; a tile with more walks per word)

// loop length of canonical seed e: len[e], or counted along next when it is the escape
// (a loop of >= kLenEsc entries)
__device__ __forceinline__ uint32_t loop_len(const uint8_t* __restrict__ len, const hid* __restrict__ next, hid e) {
  uint32_t n = len[e];
  if (n == kLenEsc) {
    n = 1;
    for (hid x = next[e]; x != e; x = next[x]) ++n;  // (the loop closed when its seed was set)
  }
  return n;
}

__global__ void __launch_bounds__(kEmitThreads)
    k_emit(int64_t T, int64_t n_words, const uint32_t* __restrict__ C, const uint8_t* __restrict__ len,
           const uint32_t* __restrict__ tb, const int32_t* __restrict__ wlen, const int32_t* __restrict__ origin,
           const hid* __restrict__ next,
           hid* __restrict__ seeds, uint32_t* __restrict__ offsets, int64_t offsets_cap, int32_t* __restrict__ loops,
           int64_t loops_cap, DevCounters* ctr) {
  pdl_enter();
  __shared__ hid qe[kEmitQ];
  __shared__ uint32_t qo[kEmitQ];
  __shared__ int32_t wbase[kEmitWords];
  __shared__ int32_t chunk[kEmitThreads / 32 + 1];
  __shared__ int32_t npoly;
  __shared__ uint32_t pbase[2];
  if (ctr->status) return;
  const int32_t P = ctr->P;
  const uint32_t L = ctr->L;
  if ((int64_t)P + 1 > offsets_cap || (int64_t)L > loops_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_status(ctr, ST_CAPACITY);
    return;
  }
  const int64_t blk = sched_tile(blockIdx.x, gridDim.x);
  const int64_t tile = blk / kEmitSub;
  const int part = (int)(blk - tile * kEmitSub);
  const int64_t wt = tile * kEmitTileWords + (int64_t)part * kEmitWords;  // first word of the part
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {  // the part's bases: the tile's + the tile's earlier words (polygons, loop entries)
    int pc = 0, lc = 0;
    for (int k = lane; k < part * kEmitWords; k += 32) {
      const int64_t ww = tile * kEmitTileWords + k;
      if (ww < n_words) {
        pc += __popc(C[ww]);
        lc += wlen[ww];
      }
    }
    pc = __reduce_add_sync(0xffffffffu, pc);
    lc = __reduce_add_sync(0xffffffffu, lc);
    if (lane == 0) {
      pbase[0] = tb[2 * tile] + (uint32_t)pc;
      pbase[1] = tb[2 * tile + 1] + (uint32_t)lc;
    }
  }
  if (warp == 0) {  // per-word exclusive prefix of the canonical-seed count
    constexpr int kWPL = kEmitWords / 32;  // 3
    int cp[kWPL], sp = 0;
#pragma unroll
    for (int k = 0; k < kWPL; ++k) {
      const int64_t ww = wt + kWPL * lane + k;
      cp[k] = ww < n_words ? __popc(C[ww]) : 0;
      sp += cp[k];
    }
    int ip = sp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ip, o);
      if (lane >= o) ip += a;
    }
    int bp = ip - sp;
#pragma unroll
    for (int k = 0; k < kWPL; ++k) {
      wbase[kWPL * lane + k] = bp;
      bp += cp[k];
    }
    if (lane == 31) npoly = ip;
  }
  __syncthreads();
  const int np = npoly;
  const uint32_t rbase = pbase[0], obase = pbase[1];
  if (np > kEmitQ) {  // (dense tile) one thread per word walks its polygons in order
    for (int wl = tid; wl < kEmitWords && wt + wl < n_words; wl += kEmitThreads) {
      // offset of the word's first polygon: tile base + lengths of the earlier polygons
      uint32_t o = obase;
      for (int64_t ww = wt; ww < wt + wl; ++ww)
        for (uint32_t b = C[ww]; b; b &= b - 1) o += loop_len(len, next, (hid)(ww * 32 + __ffs(b) - 1));
      uint32_t r = rbase + wbase[wl];
      for (uint32_t b = C[wt + wl]; b; b &= b - 1, ++r) {
        const hid e = (hid)((wt + wl) * 32 + __ffs(b) - 1);
        const int32_t n = (int32_t)loop_len(len, next, e);
        seeds[r] = e;
        offsets[r] = o;
        hid x = e;
        int32_t* dst = loops + o;  // (a pointer walk: unsigned o + i would be re-extended every step)
        for (int32_t i = 0; i < n; ++i, x = next[x]) dst[i] = origin[x];
        o += n;
      }
    }
  } else {
    // expand the seeds into the queue (rank order), then gather their loop lengths, one
    // per thread (independent loads instead of a chain per word)
    for (int wl = tid; wl < kEmitWords && wt + wl < n_words; wl += kEmitThreads) {
      int p = wbase[wl];
      for (uint32_t b = C[wt + wl]; b; b &= b - 1, ++p) qe[p] = (hid)((wt + wl) * 32 + __ffs(b) - 1);
    }
    __syncthreads();
    for (int i = tid; i < np; i += kEmitThreads) qo[i] = loop_len(len, next, qe[i]);
    __syncthreads();
    // exclusive scan of the lengths: thread t owns queue entries [t*per, (t+1)*per)
    const int per = (np + kEmitThreads - 1) / kEmitThreads;
    const int q0 = tid * per, q1 = min(q0 + per, np);
    int sum = 0;
    for (int i = q0; i < q1; ++i) sum += (int)qo[i];
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (lane == 31) chunk[warp] = inc;
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int k = 0; k < kEmitThreads / 32; ++k) { const int v = chunk[k]; chunk[k] = acc; acc += v; }
    }
    __syncthreads();
    // (tile-local sums fit int; the tile base may exceed 2^31: unsigned from here)
    uint32_t run = obase + (uint32_t)(chunk[warp] + inc - sum);
    for (int i = q0; i < q1; ++i) { const uint32_t n = qo[i]; qo[i] = run; run += n; }
    if (q1 == np && q0 < q1) chunk[kEmitThreads / 32] = (int32_t)(run - obase);  // end of the tile's last loop
    __syncthreads();
    const uint32_t run_end = obase + (uint32_t)chunk[kEmitThreads / 32];
    // one polygon per thread
    for (int i = tid; i < np; i += kEmitThreads) {
      const hid e = qe[i];
      const uint32_t o = qo[i];
      const int32_t n = (int32_t)((i + 1 < np ? qo[i + 1] : run_end) - o);
      seeds[rbase + i] = e;
      offsets[rbase + i] = o;
      hid x = e;
      int32_t* dst = loops + o;  // (a pointer walk: unsigned o + k would be re-extended every step)
      for (int32_t k = 0; k < n; ++k, x = next[x]) dst[k] = origin[x];
    }
  }
  if (blk == (int64_t)gridDim.x - 1 && tid == 0) offsets[P] = L;  // (the last part of the last tile)
}

__global__ void k_prev(int64_t T, const hid* __restrict__ next, const uint32_t* __restrict__ F1,
                       hid* __restrict__ prev, DevCounters* ctr) {
  pdl_enter();
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int64_t H = T3 + ctr->n_border;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < H; e += (int64_t)gridDim.x * blockDim.x) {
    const hid ei = (hid)e;
    if (e >= T3 || bit_of(F1, ei)) prev[next[ei]] = ei;
    else prev[ei] = prev_in(ei);
  }
}

int launch_extract(Ctx* c, uint32_t* offsets, int64_t offsets_cap, int32_t* loops, int64_t loops_cap,
                   hid* prev, cudaStream_t s) {
  int n = 0;
  prof_mark(s, "k_extract");
  if (loops) {
    const int64_t tiles = (c->T + kBuildTileTris - 1) / kBuildTileTris;
    launch_k(k_emit, (unsigned)(tiles * kEmitSub), kEmitThreads, 0, s, c->T, c->n_words, c->C, c->len, c->tbase, c->wlen,
             c->origin, c->next,
                                                   c->seeds, offsets ? offsets : c->offsets,
                                                   offsets ? offsets_cap : c->T + 1, loops, loops_cap, c->ctr);
    ++n;
  }
  if (prev) {
    launch_k(k_prev, 148 * 16, 256, 0, s, c->T, c->next, c->F1, prev, c->ctr);
    ++n;
  }
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? n : -1;
}

}  // namespace polylla
