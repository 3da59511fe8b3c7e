// check.cu -- exact non-manifold-edge detection (SPEC.md L49 NonManifoldEdge: "an
// undirected edge in more than two triangles, or twice in one direction").
//
// The tiled build (build.cu) detects it exactly when all copies of an edge fall in one
// build tile, and among the cross-tile leftovers.  A copy that pairs inside its tile
// while another copy sits in another tile is not seen there (R20).  This
// opt-in pass (polylla_check_manifold) closes the gap: every interior half-edge looks up
// its UNDIRECTED key {origin, target} in a global hash; the first copy claims a slot, a
// second copy in the opposite direction marks it paired, and a second copy in the same
// direction or any third copy raises ST_NONMANIFOLD_EDGE (SPEC.md L49's rule, exactly).
//
// Scratch: the leftover-key region (24T bytes), dead once the build has ranked its
// border half-edges; slots hold a half-edge id plus a paired flag (the key is re-read
// from origin[]); at most (3T + B) / 2 <= 3T distinct keys in >= 3T slots.
#include "internal.cuh"

namespace polylla {

constexpr uint32_t kPaired = 0x80000000u;  // flag in the slots (half-edge ids < 2^31: see polylla_check_manifold)

__global__ void k_dup_clear(uint32_t* slots, int64_t cap) {
  uint4* s4 = reinterpret_cast<uint4*>(slots);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap / 4; i += (int64_t)gridDim.x * blockDim.x)
    s4[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
}

__global__ void k_dup_insert(int64_t T, const int32_t* __restrict__ origin, uint32_t* slots, int64_t cap,
                             DevCounters* ctr) {
  // (runs whatever the status: it only reads origin[], written in full by k_tile, and an
  // edge error outranks the vertex error the border chaining may have raised for it)
  const int64_t T3 = 3 * T;
  const uint32_t mask = (uint32_t)(cap - 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < T3; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ei = (int32_t)e;
    const uint32_t o = (uint32_t)origin[ei], t = (uint32_t)origin[next_in(ei)];
    uint32_t h = mix32(min(o, t), max(o, t)) & mask;
    for (uint32_t probe = 0; probe <= mask; ++probe, h = (h + 1) & mask) {
      uint32_t s = slots[h];
      if (s == kEmpty) {
        s = atomicCAS(&slots[h], kEmpty, (uint32_t)ei);
        if (s == kEmpty) break;  // first copy of the edge
      }
      const int32_t si = (int32_t)(s & ~kPaired);
      const uint32_t so = (uint32_t)origin[si], st = (uint32_t)origin[next_in(si)];
      if (so == o && st == t) {  // the same directed edge twice
        raise_status(ctr, ST_NONMANIFOLD_EDGE);
        break;
      }
      if (so == t && st == o) {  // the opposite copy: pair it, unless it already was (a third copy)
        if ((s & kPaired) || atomicCAS(&slots[h], s, s | kPaired) != s) raise_status(ctr, ST_NONMANIFOLD_EDGE);
        break;
      }
    }
  }
}

int launch_check_manifold(Ctx* c, cudaStream_t s) {
  // capacity: the largest power of two <= 6T slots of 4 bytes (24T bytes), >= 3T keys
  int64_t cap = 4;
  while (2 * cap <= 6 * c->T) cap <<= 1;
  uint32_t* slots = reinterpret_cast<uint32_t*>(c->left_key);
  prof_mark(s, "k_check_manifold");
  k_dup_clear<<<148 * 8, 256, 0, s>>>(slots, cap);
  k_dup_insert<<<148 * 8, 256, 0, s>>>(c->T, c->origin, slots, cap, c->ctr);
  prof_end(s);
  return cudaGetLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace polylla
