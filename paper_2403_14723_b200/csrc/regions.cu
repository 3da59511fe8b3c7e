// regions.cu -- per-triangle polygon ids and terminal-edge-region ids (SURVEY.md §8(f)
// NEXT-4).  (1) Post-repair: the output polygons
// of PAPER.md L113 / L579 as unions of triangles, i.e. the terminal-edge regions of
// PAPER.md L76-L128 after the barrier repair.  A polygon's triangles are the piece of
// triangles connected across its non-frontier (F1 = 0) edges; its loop bounds the piece.
//   poly_of_tri[t] = min { p : the loop of polygon p bounds the piece of t }
// (a piece has several loops only around a hole of the mesh).
// (2) Pre-repair: the terminal-edge regions of PAPER.md Defs. 1-2 (L121-128), the Lepp
// partition that the data-parallel Lepp of PAPER.md L76 refines: the pieces of triangles
// connected across non-frontier edges of F0 (the frontier before the repair), labelled by
// their smallest triangle id.
// GPU: lock-free union-find over the non-frontier interior edges (hook the larger root
// under the smaller with CAS, path halving in find; per tile in shared memory first), then every polygon's canonical seed
// (an interior half-edge of its loop, whose triangle lies in the piece) takes the min over
// its root, and every triangle reads its root's value.
#include "internal.cuh"

namespace polylla {

// global parents: relaxed GPU-scope atomic loads/stores (served by L2, like ld.cg)
__device__ __forceinline__ int32_t ld_rlx_g(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_rlx_g(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v));
}

__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t x) {
  // path halving; parents only ever decrease (a root is hooked under a smaller root), so a
  // racy halving store still points into the same tree
  while (true) {
    const int32_t p = ld_rlx_g(parent + x);
    if (p == x) return x;
    const int32_t g = ld_rlx_g(parent + p);
    if (p == g) return p;
    st_rlx_g(parent + x, g);
    x = g;
  }
}

// shared-memory parents: relaxed CTA-scope atomic loads/stores (plain LDS/STS in SASS; the
// halving stores race with the hooks' CAS by design, so they are atomics in the PTX memory
// model, not data races)
__device__ __forceinline__ int32_t ld_rlx_s(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ void st_rlx_s(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.cta.shared.s32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v));
}
__device__ __forceinline__ int32_t uf_find_s(int32_t* p, int32_t x) {
  while (true) {
    const int32_t q = ld_rlx_s(p + x);
    if (q == x) return x;
    const int32_t g = ld_rlx_s(p + q);
    if (q == g) return q;
    st_rlx_s(p + x, g);
    x = g;
  }
}

// One block per build tile of kBuildTileTris triangles: the unions whose two triangles lie
// in the tile (most of them: triangles come in spatial order) in shared memory, then the
// tile's forest goes out as the initial global parents (a local root keeps the smallest id
// of its set, so parents still only decrease).
#ifndef POLYLLA_UF_THREADS
#define POLYLLA_UF_THREADS 512  // measured 256 / 384 / 512 / 1024 on config 3: 512 best (0.46 ms)
#endif
constexpr int kUfTile = kBuildTileTris, kUfThreads = POLYLLA_UF_THREADS;
static_assert(3 * kUfTile % kUfThreads == 0, "half-edges per thread");
__global__ void __launch_bounds__(kUfThreads) k_uf_local(int64_t T, const hid* __restrict__ twin,
                                                  const uint32_t* __restrict__ F1, int32_t* __restrict__ parent,
                                                  int32_t* __restrict__ slot, hid* __restrict__ cross,
                                                  DevCounters* ctr) {
  __shared__ int32_t p[kUfTile];
  if (ctr->status) return;
  const int64_t t0 = (int64_t)blockIdx.x * kUfTile;
  const int nt = T - t0 < kUfTile ? (int)(T - t0) : kUfTile;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) p[i] = i;
  __syncthreads();
  const hid e0 = (hid)(3 * t0);
  constexpr int kIt = 3 * kUfTile / kUfThreads;
  hid tws[kIt];
#pragma unroll
  // a thread takes kIt consecutive half-edges (4 triangles): neighbouring lanes then unite
  // different pieces (interleaved lanes all hook the same few roots and retry their CAS)
  for (int k = 0; k < kIt; ++k) {  // all of the thread's loads first (independent)
    const int j = threadIdx.x * kIt + k;
    tws[k] = j < 3 * nt && !bit_of(F1, e0 + j) ? __ldcs(twin + e0 + j) : kNoHe;
  }
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const int j = threadIdx.x * kIt + k;
    const hid e = e0 + j, tw = tws[k];
    if (cross && tw != kNoHe && tw > e && tw >= e0 + 3 * nt) {  // (grid tiling) a pair to the hook list
      const uint32_t m = __activemask();
      const int leader = __ffs(m) - 1, rank = __popc(m & ((1u << (threadIdx.x & 31)) - 1));
      uint32_t b = 0;
      if ((int)(threadIdx.x & 31) == leader) b = atomicAdd(&ctr->n_cross, (uint32_t)__popc(m));
      cross[__shfl_sync(m, b, leader) + rank] = e;
      continue;
    }
    if (tw < e || tw >= e0 + 3 * nt) continue;  // frontier (kNoHe); once per pair; cross-tile pairs: k_uf_hook
    int32_t a = j / 3, b = (int32_t)((tw - e0) / 3);
    while (true) {
      a = uf_find_s(p, a);
      b = uf_find_s(p, b);
      if (a == b) break;
      if (a < b) { const int32_t s = a; a = b; b = s; }
      if (atomicCAS(p + a, a, b) == a) break;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    parent[t0 + i] = (int32_t)t0 + uf_find_s(p, i);
    slot[t0 + i] = INT32_MAX;
  }
}

// the cross-tile pairs: both halves of each are in k_tile's leftover lists (tile t:
// entries [3 * kBuildTileTris * t, + cnt_ld[2t]) of left_e); one block per tile segment
__global__ void k_uf_hook(int64_t ntiles, const int32_t* __restrict__ cnt_ld, const hid* __restrict__ left_e,
                          const hid* __restrict__ twin, const uint32_t* __restrict__ F1, int32_t* parent,
                          const DevCounters* ctr) {
  if (ctr->status) return;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int32_t n = cnt_ld[2 * tile];
    const int64_t base = 3 * (int64_t)kBuildTileTris * tile;
    for (int32_t k = threadIdx.x; k < n; k += blockDim.x) {
      const hid e = left_e[base + k];
      if (bit_of(F1, e)) continue;  // frontier (incl. the border ones)
      const hid tw = twin[e];
      if (tw < e) continue;  // once per pair, from its lower half
      int32_t a = (int32_t)(e / 3), b = (int32_t)(tw / 3);
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

// (grid tiling) the pairs crossing the union-find tiles, listed by k_uf_local: the build
// tiles are 2-D patches there, so their leftover lists miss pairs that k_uf_local's
// contiguous tiles split
__global__ void k_uf_hook_list(const hid* __restrict__ cross, const hid* __restrict__ twin, int32_t* parent,
                               const DevCounters* ctr) {
  if (ctr->status) return;
  const uint32_t n = ctr->n_cross;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const hid e = cross[i];
    int32_t a = (int32_t)(e / 3), b = (int32_t)(twin[e] / 3);
    while (true) {
      a = uf_find(parent, a);
      b = uf_find(parent, b);
      if (a == b) break;
      if (a < b) { const int32_t s = a; a = b; b = s; }
      if (atomicCAS(parent + a, a, b) == a) break;
    }
  }
}

__global__ void k_uf_seed(const hid* __restrict__ seeds, int32_t* parent, int32_t* __restrict__ slot,
                          const DevCounters* ctr) {
  if (ctr->status) return;
  const int32_t P = ctr->P;
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x)
    atomicMin(slot + uf_find(parent, (int32_t)(seeds[p] / 3)), p);
}

__global__ void k_uf_out(int64_t T, int32_t* parent, const int32_t* __restrict__ slot, int32_t* __restrict__ out,
                         const DevCounters* ctr) {
  const bool bad = ctr->status != 0;  // (e.g. a capacity error: no seeds were written) -> all -1
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    if (bad) {
      out[t] = -1;
      continue;
    }
    const int32_t v = slot[uf_find(parent, (int32_t)t)];
    out[t] = v == INT32_MAX ? -1 : v;  // -1: a piece without a loop (not reachable on valid output)
  }
}

// pre-repair terminal-edge regions: every triangle reads its root, which is the smallest
// triangle id of its set (roots only ever hook under smaller roots)
__global__ void k_uf_roots(int64_t T, int32_t* parent, int32_t* __restrict__ out, const DevCounters* ctr) {
  const bool bad = ctr->status != 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = bad ? -1 : uf_find(parent, (int32_t)t);
}

// out[t]: post-repair polygon index (F1 pieces, mode 0) or pre-repair terminal-edge region
// label = smallest triangle id of the region (F0 pieces, mode 1)
int launch_regions(Ctx* c, int32_t* out, int mode, cudaStream_t s) {
  // scratch: the leftover-key region (24 B per interior triangle slot, dead after the build)
  int32_t* parent = reinterpret_cast<int32_t*>(c->left_key);
  int32_t* slot = parent + c->T;
  const uint32_t* F = mode == 1 ? c->F0 : c->F1;
  const unsigned g = 148 * 8;
  prof_mark(s, mode == 1 ? "k_regions_pre" : "k_regions");
  hid* cross = c->tiling.mode != kTileContig ? reinterpret_cast<hid*>(slot + c->T) : nullptr;  // (16T bytes left of the 24T scratch)
  if (cross) cudaMemsetAsync(&c->ctr->n_cross, 0, 4, s);
  k_uf_local<<<(unsigned)((c->T + kUfTile - 1) / kUfTile), kUfThreads, 0, s>>>(c->T, c->twin, F, parent, slot,
                                                                                 cross, c->ctr);
  const int64_t tiles = (c->T + kUfTile - 1) / kUfTile;
  if (cross)
    k_uf_hook_list<<<148 * 8, 256, 0, s>>>(cross, c->twin, parent, c->ctr);
  else
    k_uf_hook<<<(unsigned)tiles, 256, 0, s>>>(tiles, c->cnt_ld, c->left_e, c->twin, F, parent, c->ctr);
  if (mode == 1) {
    k_uf_roots<<<g, 256, 0, s>>>(c->T, parent, out, c->ctr);
  } else {
    k_uf_seed<<<g, 256, 0, s>>>(c->seeds, parent, slot, c->ctr);
    k_uf_out<<<g, 256, 0, s>>>(c->T, parent, slot, out, c->ctr);
  }
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? (mode == 1 ? 3 : 4) : -1;
}

}  // namespace polylla
