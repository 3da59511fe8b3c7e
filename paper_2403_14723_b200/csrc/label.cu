// label.cu -- label phase (Alg. 8 "LabelFrontierEdges", Alg. 9
// "LabelSeedEdges") fused with the unlink rewire (Alg. 11 "Change attributes",
// PAPER.md L739-775) and barrier-tip detection -- the part k_tile (build.cu) could not
// finish inside its tile.  Per half-edge e:
//   F[e] = border(twin e) or (not L[e] and not L[twin e])                 (Alg. 8, R15)
//   S[e] = L[e] and (border(twin e) or (L[twin e] and e < twin e))        (Alg. 9, R8)
//   frontier e: x <- next_in(e); while not F[x]: x <- next_in(twin x);     (Alg. 11, R1/R3)
//               next[e] <- x; a barrier tip iff x == twin(e)              (R4)
//   otherwise : next[e] <- next_in(e)                                     (R14)
// L[x] is recomputed on the fly from Lcode (T bytes, L2-resident) so the walk does not
// depend on other threads' F bits.  The rewire is in place: a thread writes only
// next[e] of its own e and reads only twin/Lcode.
#include "internal.cuh"

namespace polylla {

#ifndef POLYLLA_FIX_THREADS
#define POLYLLA_FIX_THREADS 384  // 128 / 256 / 384 / 512 measured: 384 best on config 3
#endif
constexpr int kLabelThreads = POLYLLA_FIX_THREADS;

__device__ __forceinline__ bool is_longest(const uint8_t* __restrict__ lcode, hid x) {
  const hid f = x / 3u;
  return (hid)lcode[f] == x - 3u * f;
}

// One thread per half-edge deferred by k_tile (its twin, or a twin met by its rotation
// walk, lies outside the build tile).  Same computation as k_tile's P4, on the global
// arrays; bit-vector words (F0, F1, S, and TB / SDB: tips and seeds for the generate
// phase) are completed with atomicOr.  The deferred half-edges of tile t are entries
// [3 * 2048 * t, + cnt_ld[2t + 1]) of def_e; one block per tile segment.
__global__ void __launch_bounds__(kLabelThreads)
    k_label_fixup(int64_t T, int64_t ntiles, const Tiling tl, const int32_t* __restrict__ cnt_ld, const hid* __restrict__ def_e,
                  const hid* __restrict__ twin, const uint8_t* __restrict__ lcode, hid* __restrict__ next,
                  uint32_t* __restrict__ F0, uint32_t* __restrict__ F1, uint32_t* __restrict__ S,
                  uint32_t* __restrict__ TB, uint32_t* __restrict__ SDB, DevCounters* ctr) {
  pdl_enter();
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int lane = threadIdx.x & 31;
  for (int64_t it = blockIdx.x; it < ntiles; it += gridDim.x) {
    const int64_t tile = sched_tile(it, ntiles);
    const int32_t n = cnt_ld[2 * tile + 1];
    const int64_t seg = tile_geom(tl, T, tile).seg;
    for (int32_t base = 0; base < n; base += kLabelThreads) {  // warp-uniform trip count
      const int32_t i = base + threadIdx.x;
      bool tip = false, walk_err = false, sd = false, fr = false;
      hid e = kNoHe;
      if (i < n) {
        e = def_e[seg + i];
        const hid t = twin[e];
        const bool tb = t >= T3;
        const bool Le = is_longest(lcode, e);
        const bool Lt = !tb && is_longest(lcode, t);
        fr = tb || (!Le && !Lt);
        sd = Le && (tb || (Lt && e < t));
        hid nx = next_in(e);
        if (fr) {
          hid x = nx;
          for (int64_t steps = 0;; ++steps) {  // bound: a rotation has <= deg(v) <= 3T steps
            const hid tx = twin[x];
            if (tx >= T3) break;                                         // border edge: frontier
            if (!is_longest(lcode, x) && !is_longest(lcode, tx)) break;  // frontier edge
            x = next_in(tx);                                             // cross the edge (sweep_out)
            if (steps > T3) { walk_err = true; break; }
          }
          nx = x;
          tip = (x == t);
        }
        next[e] = nx;
      }
      // bit-vector words: deferred entries are in ascending order per tile, so
      // neighbouring lanes usually share a word -> one atomicOr per distinct word
      const uint32_t word = e != kNoHe ? (uint32_t)(e >> 5) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, word);
      const uint32_t bit = e != kNoHe ? 1u << (e & 31) : 0u;
      const uint32_t fbits = __reduce_or_sync(peers, fr ? bit : 0u);
      const uint32_t sbits = __reduce_or_sync(peers, sd ? bit : 0u);
      const uint32_t tbits = __reduce_or_sync(peers, tip ? bit : 0u);
      if (e != kNoHe && lane == __ffs(peers) - 1) {
        if (fbits) { atomicOr(&F0[word], fbits); atomicOr(&F1[word], fbits); }
        if (sbits) { atomicOr(&S[word], sbits); atomicOr(&SDB[word], sbits); }  // seeds found here: global walk
        if (tbits) atomicOr(&TB[word], tbits);
      }
      if (walk_err) raise_status(ctr, ST_WALK);
    }
  }
}

constexpr int kFixBlocksPerSM = 4096 / kLabelThreads;  // a grid of 2 resident waves

int launch_label(Ctx* c, cudaStream_t s) {
  const int64_t tiles = c->tiling.ntiles;
  prof_mark(s, "k_label_fixup");
  launch_k(k_label_fixup, (unsigned)(tiles < 148 * kFixBlocksPerSM ? tiles : 148 * kFixBlocksPerSM), kLabelThreads, 0, s, 
      c->T, tiles, c->tiling, c->cnt_ld, c->def_e, c->twin, c->lcode, c->next, c->F0, c->F1, c->S, c->TB, c->SDB, c->ctr);
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace polylla
