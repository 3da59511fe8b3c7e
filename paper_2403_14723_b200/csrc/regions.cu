// regions.cu -- per-triangle polygon ids: the output polygons
// of PAPER.md L113 / L579 as unions of triangles, i.e. the terminal-edge regions of
// PAPER.md L76-L128 after the barrier repair.  A polygon's triangles are the piece of
// triangles connected across its non-frontier (F1 = 0) edges; its loop bounds the piece.
//   poly_of_tri[t] = min { p : the loop of polygon p bounds the piece of t }
// (a piece has several loops only around a hole of the mesh).
// GPU: lock-free union-find over the non-frontier interior edges (hook the larger root
// under the smaller with CAS, path halving in find), then every polygon's canonical seed
// (an interior half-edge of its loop, whose triangle lies in the piece) takes the min over
// its root, and every triangle reads its root's value.
#include "internal.cuh"

namespace polylla {

__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t x) {
  // path halving; parents only ever decrease (a root is hooked under a smaller root), so a
  // racy halving store still points into the same tree
  while (true) {
    const int32_t p = __ldcg(parent + x);
    if (p == x) return x;
    const int32_t g = __ldcg(parent + p);
    if (p == g) return p;
    __stcg(parent + x, g);
    x = g;
  }
}

__global__ void k_uf_init(int64_t T, int32_t* __restrict__ parent, int32_t* __restrict__ slot) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    parent[t] = (int32_t)t;
    slot[t] = INT32_MAX;
  }
}

// one thread per word of 32 interior half-edges: every non-frontier e < twin(e) unites
// its two triangles (a non-frontier edge is interior on both sides)
__global__ void k_uf_hook(int64_t T, int64_t n_words, const int32_t* __restrict__ twin, const uint32_t* __restrict__ F1,
                          int32_t* parent, const DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = w * 32;
    uint32_t m = ~F1[w];
    if (T3 - e0 < 32) m &= (1u << (T3 - e0)) - 1u;
    for (; m; m &= m - 1) {
      const int32_t e = (int32_t)(e0 + __ffs(m) - 1);
      const int32_t tw = twin[e];
      if (tw < e) continue;  // the pair is united once, from its lower half
      int32_t a = e / 3, b = tw / 3;
      while (true) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) break;
        if (a < b) { const int32_t s = a; a = b; b = s; }  // hook the larger root a under b
        if (atomicCAS(parent + a, a, b) == a) break;
      }
    }
  }
}

__global__ void k_uf_seed(const int32_t* __restrict__ seeds, int32_t* parent, int32_t* __restrict__ slot,
                          const DevCounters* ctr) {
  if (ctr->status) return;
  const int32_t P = ctr->P;
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x)
    atomicMin(slot + uf_find(parent, seeds[p] / 3), p);
}

__global__ void k_uf_out(int64_t T, int32_t* parent, const int32_t* __restrict__ slot, int32_t* __restrict__ out,
                         const DevCounters* ctr) {
  if (ctr->status) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = slot[uf_find(parent, (int32_t)t)];
    out[t] = v == INT32_MAX ? -1 : v;  // -1: a piece without a loop (not reachable on valid output)
  }
}

int launch_regions(Ctx* c, int32_t* poly_of_tri, cudaStream_t s) {
  // scratch: the leftover-key region (24 B per interior triangle slot, dead after generate)
  int32_t* parent = reinterpret_cast<int32_t*>(c->left_key);
  int32_t* slot = parent + c->T;
  const unsigned g = 148 * 8;
  prof_mark(s, "k_regions");
  k_uf_init<<<g, 256, 0, s>>>(c->T, parent, slot);
  k_uf_hook<<<g, 256, 0, s>>>(c->T, c->n_words, c->twin, c->F1, parent, c->ctr);
  k_uf_seed<<<g, 256, 0, s>>>(c->seeds, parent, slot, c->ctr);
  k_uf_out<<<g, 256, 0, s>>>(c->T, parent, slot, poly_of_tri, c->ctr);
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? 4 : -1;
}

}  // namespace polylla
