// extract.cu -- polygon extraction ("the seed list is used to rebuild
// each polygon of the output mesh using the next ... queries"), moved on-device:
//   loops[offsets[p] + i] = origin[x_i], x_0 = seeds[p], x_{i+1} = next[x_i]   (CSR)
// plus the optional prev array: the inverse of next on frontier and border
// half-edges (their next is a permutation of them), prev_in on the others.
#include "internal.cuh"

namespace polylla {

__global__ void k_extract(const int32_t* __restrict__ seeds, const int32_t* __restrict__ offs_in,
                          const int32_t* __restrict__ origin, const int32_t* __restrict__ next,
                          int32_t* __restrict__ offsets, int64_t offsets_cap, int32_t* __restrict__ loops,
                          int64_t loops_cap, DevCounters* ctr) {
  if (ctr->status) return;
  const int32_t P = ctr->P;
  const int32_t L = ctr->L;
  if ((int64_t)P + 1 > offsets_cap || (int64_t)L > loops_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_status(ctr, ST_CAPACITY);
    return;
  }
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p <= P; p += gridDim.x * blockDim.x) {
    const int32_t o = offs_in[p];
    if (offsets) offsets[p] = o;
    if (p == P) break;
    const int32_t n = offs_in[p + 1] - o;
    int32_t x = seeds[p];
    for (int32_t i = 0; i < n; ++i) {
      loops[o + i] = origin[x];
      x = next[x];
    }
  }
}

__global__ void k_prev(int64_t T, const int32_t* __restrict__ next, const uint32_t* __restrict__ F1,
                       int32_t* __restrict__ prev, DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  const int64_t H = T3 + ctr->n_border;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < H; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ei = (int32_t)e;
    if (e >= T3 || bit_of(F1, ei)) prev[next[ei]] = ei;
    else prev[ei] = prev_in(ei);
  }
}

int launch_extract(Ctx* c, int32_t* offsets, int64_t offsets_cap, int32_t* loops, int64_t loops_cap,
                   int32_t* prev, cudaStream_t s) {
  int n = 0;
  prof_mark(s, "k_extract");
  if (loops) k_extract<<<148 * 8, 256, 0, s>>>(c->seeds, c->offsets, c->origin, c->next, offsets, offsets_cap, loops, loops_cap,
                                    c->ctr), ++n;
  if (prev) {
    k_prev<<<148 * 16, 256, 0, s>>>(c->T, c->next, c->F1, prev, c->ctr);
    ++n;
  }
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? n : -1;
}

}  // namespace polylla
