// label.cu -- label phase (Alg. 8 "LabelFrontierEdges", Alg. 9
// "LabelSeedEdges") fused with the unlink rewire (Alg. 11 "Change attributes",
// PAPER.md L739-775) and barrier-tip detection.
//
// One thread per interior half-edge e (coalesced over e):
//   F[e] = border(twin e) or (not L[e] and not L[twin e])                 (Alg. 8, R15)
//   S[e] = L[e] and (border(twin e) or (L[twin e] and e < twin e))        (Alg. 9, R8)
//   frontier e: x <- next_in(e); while not F[x]: x <- next_in(twin x);     (Alg. 11, R1/R3)
//               next[e] <- x; a barrier tip iff x == twin(e)              (R4)
//   otherwise : next[e] <- next_in(e)                                     (R14)
// L[x] is recomputed on the fly from Lcode (T bytes, L2-resident) so the walk does not
// depend on other threads' F bits; F/S words are produced with warp ballots (a warp
// covers 32 consecutive half-edges = one bit-vector word).  The rewire is in place:
// a thread writes only next[e] of its own e and reads only twin/Lcode.
#include "internal.cuh"

namespace polylla {

constexpr int kLabelThreads = 256;

__device__ __forceinline__ bool is_longest(const uint8_t* __restrict__ lcode, int32_t x) {
  const int32_t f = x / 3;
  return (int32_t)lcode[f] == x - 3 * f;
}

__global__ void __launch_bounds__(kLabelThreads)
    k_label_rewire(int64_t T, const int32_t* __restrict__ twin, const uint8_t* __restrict__ lcode,
                   int32_t* __restrict__ next, uint32_t* __restrict__ F0, uint32_t* __restrict__ F1,
                   uint32_t* __restrict__ S, int32_t* __restrict__ tips, DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int64_t e64 = (int64_t)blockIdx.x * kLabelThreads + threadIdx.x;
  const bool valid = e64 < T3;
  const int32_t e = (int32_t)e64;
  bool fr = false, sd = false, tip = false;
  bool walk_err = false;
  if (valid) {
    const int32_t t = twin[e];
    const bool tb = t >= T3;
    const bool Le = is_longest(lcode, e);
    const bool Lt = !tb && is_longest(lcode, t);
    fr = tb || (!Le && !Lt);
    sd = Le && (tb || (Lt && e < t));
    int32_t nx = next_in(e);
    if (fr) {
      int32_t x = nx;
      for (int steps = 0;; ++steps) {
        const int32_t tx = twin[x];
        if (tx >= T3) break;                                     // border edge: frontier
        if (!is_longest(lcode, x) && !is_longest(lcode, tx)) break;  // frontier edge
        x = next_in(tx);                                         // cross the edge (sweep_out)
        if (steps > kWalkBound) { walk_err = true; break; }
      }
      nx = x;
      tip = (x == t);
    }
    next[e] = nx;
  }
  const uint32_t fw = __ballot_sync(0xffffffffu, fr);
  const uint32_t sw = __ballot_sync(0xffffffffu, sd);
  const uint32_t tm = __ballot_sync(0xffffffffu, tip);
  const int lane = threadIdx.x & 31;
  const int64_t wbase = e64 - lane;
  if (lane == 0 && wbase < T3) {
    F0[wbase >> 5] = fw;
    F1[wbase >> 5] = fw;
    S[wbase >> 5] = sw;
  }
  if (tm) {
    int pos = 0;
    if (lane == 0) pos = atomicAdd(&ctr->n_tips, __popc(tm));
    pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(tm & ((1u << lane) - 1));
    if (tip) tips[pos] = e;
  }
  if (walk_err) raise_status(ctr, ST_WALK);
}

int launch_label(Ctx* c, cudaStream_t s) {
  const int64_t blocks = (3 * c->T + kLabelThreads - 1) / kLabelThreads;
  prof_mark(s, "k_label_rewire");
  k_label_rewire<<<(unsigned)blocks, kLabelThreads, 0, s>>>(c->T, c->twin, c->lcode, c->next, c->F0, c->F1, c->S,
                                                           c->tips, c->ctr);
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace polylla
