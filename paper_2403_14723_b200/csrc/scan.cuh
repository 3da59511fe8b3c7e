// scan.cuh -- order-preserving compaction of a bit-vector ("scan and
// compact seed edges array"), reduce-then-scan in three launches:
//   1. k_scan_reduce : per block of kScanWords words, (#set bits, Op::word_aux = dense
//                      per-word sum of aux, extra per-word sum) -> 3 block sums;
//   2. k_scan_top    : one block, exclusive scan of the block sums, totals to Op::finish;
//   3. k_scan_down   : per block, the rank and aux-prefix of every set bit -> Op::emit.
// Ranks follow ascending bit position, so the output is deterministic.  The paper
// accelerates this scan with tensor cores; here it is HBM-bound bit counting (warp
// popc + shuffles), which is what the hardware is good at for this shape.
#pragma once
#include "internal.cuh"

namespace polylla {

constexpr int kScanThreads = 256;
constexpr int kScanWPT = 8;  // words per thread
constexpr int kScanWords = kScanThreads * kScanWPT;

struct Sum3 {
  long long a, b, c;
};

__device__ __forceinline__ Sum3 warp_incl_scan(Sum3 v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long a = __shfl_up_sync(0xffffffffu, v.a, o);
    long long b = __shfl_up_sync(0xffffffffu, v.b, o);
    long long c = __shfl_up_sync(0xffffffffu, v.c, o);
    if (lane >= o) { v.a += a; v.b += b; v.c += c; }
  }
  return v;
}

// Block-wide exclusive scan; returns the exclusive prefix of this thread and writes
// the block total to *total (all threads).
__device__ __forceinline__ Sum3 block_excl_scan(Sum3 v, Sum3* total) {
  __shared__ Sum3 warp_tot[kScanThreads / 32];
  __shared__ Sum3 all;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Sum3 inc = warp_incl_scan(v);
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    Sum3 t = lane < kScanThreads / 32 ? warp_tot[lane] : Sum3{0, 0, 0};
    Sum3 ti = warp_incl_scan(t);
    if (lane < kScanThreads / 32) warp_tot[lane] = Sum3{ti.a - t.a, ti.b - t.b, ti.c - t.c};
    if (lane == kScanThreads / 32 - 1) all = ti;
  }
  __syncthreads();
  Sum3 base = warp_tot[wid];
  *total = all;
  __syncthreads();
  return Sum3{base.a + inc.a - v.a, base.b + inc.b - v.b, base.c + inc.c - v.c};
}

template <class Op>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Op op, int64_t n_words, long long* sa, long long* sb,
                                                              long long* sc) {
  if (op.skip()) return;
  const int64_t w0 = (int64_t)blockIdx.x * kScanWords;
  Sum3 v{0, 0, 0};
  // coalesced: thread t reads words w0 + t + i*kScanThreads
#pragma unroll
  for (int i = 0; i < kScanWPT; ++i) {
    const int64_t w = w0 + threadIdx.x + (int64_t)i * kScanThreads;
    if (w < n_words) {
      uint32_t bits = op.word(w);
      v.a += __popc(bits);
      v.b += op.word_aux(w, bits);  // sum of aux over the set bits of word w
      v.c += op.extra(w);
    }
  }
  Sum3 tot;
  block_excl_scan(v, &tot);
  if (threadIdx.x == 0) { sa[blockIdx.x] = tot.a; sb[blockIdx.x] = tot.b; sc[blockIdx.x] = tot.c; }
}

template <class Op>
__global__ void __launch_bounds__(kScanThreads) k_scan_top(Op op, int64_t nb, long long* sa, long long* sb,
                                                           long long* sc) {
  if (op.skip()) return;
  Sum3 carry{0, 0, 0};
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    Sum3 v = i < nb ? Sum3{sa[i], sb[i], sc[i]} : Sum3{0, 0, 0};
    Sum3 tot;
    Sum3 ex = block_excl_scan(v, &tot);
    if (i < nb) { sa[i] = carry.a + ex.a; sb[i] = carry.b + ex.b; sc[i] = carry.c + ex.c; }
    carry.a += tot.a; carry.b += tot.b; carry.c += tot.c;
  }
  if (threadIdx.x == 0) op.finish(carry.a, carry.b, carry.c);
}

template <class Op>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(Op op, int64_t n_words, const long long* sa,
                                                            const long long* sb) {
  if (op.skip()) return;
  // here thread t owns kScanWPT CONSECUTIVE words so ranks follow bit order
  const int64_t w0 = (int64_t)blockIdx.x * kScanWords + (int64_t)threadIdx.x * kScanWPT;
  uint32_t bits[kScanWPT];
  Sum3 v{0, 0, 0};
#pragma unroll
  for (int i = 0; i < kScanWPT; ++i) {
    const int64_t w = w0 + i;
    bits[i] = w < n_words ? op.word(w) : 0u;
    v.a += __popc(bits[i]);
    if (bits[i]) v.b += op.word_aux(w, bits[i]);
  }
  Sum3 tot;
  Sum3 ex = block_excl_scan(v, &tot);
  long long rank = sa[blockIdx.x] + ex.a;
  long long pre = sb[blockIdx.x] + ex.b;
#pragma unroll
  for (int i = 0; i < kScanWPT; ++i) {
    uint32_t b = bits[i];
    while (b) {
      const int k = __ffs(b) - 1;
      b &= b - 1;
      const int32_t e = (int32_t)((w0 + i) * 32 + k);
      const long long a = op.aux(e);
      op.emit(e, rank, pre);
      ++rank;
      pre += a;
    }
  }
}

template <class Op>
inline int launch_scan(const Op& op, int64_t n_words, long long* sa, long long* sb, long long* sc,
                       cudaStream_t s) {
  const int64_t nb = (n_words + kScanWords - 1) / kScanWords;
  if (nb == 0) return 0;
  k_scan_reduce<Op><<<(unsigned)nb, kScanThreads, 0, s>>>(op, n_words, sa, sb, sc);
  k_scan_top<Op><<<1, kScanThreads, 0, s>>>(op, nb, sa, sb, sc);
  k_scan_down<Op><<<(unsigned)nb, kScanThreads, 0, s>>>(op, n_words, sa, sb);
  return cudaGetLastError() == cudaSuccess ? 3 : -1;
}

}  // namespace polylla
