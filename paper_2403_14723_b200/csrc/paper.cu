// paper.cu -- the paper's own GPU kernel sequence, as an ablation.
//
// GPolylla's Algorithm runs, after the half-edge build, one kernel
// per step with one thread per element:
//   LLK  Alg. 7  "Label longest edge"        per triangle
//   LFK  Alg. 8  "Label frontier edges"      per half-edge (L638-665)
//   LSK  Alg. 9  "Label seed edges"          per half-edge (L667-691)
//   LEK  Alg. 10 "Label extra frontier edge" per VERTEX   (L696-737): count the frontier
//        edges around v; a vertex with exactly one is a barrier tip: its middle edge
//        becomes frontier and both halves seeds -- the repair done BEFORE the rewire
//   CaK  Alg. 11 "Change attributes"         per half-edge (L739-775): next and prev of
//        every frontier half-edge by rotation to the next / previous frontier half-edge
//   SFK  Alg. 12 "Search frontier edges"     per seed      (L778-810)
//   OSK  "Overwrite seeds"                   per seed      (L812-849): walk the polygon,
//        keep the minimum id as its seed
//   Scan "Scan and compact"                              (L852-858)
// with the readings of DESIGN.md (R1 rotations by the edge crossed, R5 middle edge, R6
// snapshot: LEK reads F0 and writes F1, R8/R13 seeds, R14 non-frontier keep next_in).
// Where this repo's pipeline (build.cu -> generate.cu) fuses LLK/LFK/LSK/CaK into the
// build tile, detects tips in O(1) as next == twin and repairs only around them, this
// path walks every vertex (LEK) and rotates every half-edge (CaK) as printed.  It shares
// the build (the half-edge structure) and the compaction/extraction with the main path,
// and must give bit-identical results (tests/test_gpu_paper.py).
#include "internal.cuh"

namespace polylla {

namespace {

__device__ __forceinline__ double sq_len_p(const double2* xy, int32_t o, int32_t t) {
  const double2 p = xy[o], q = xy[t];
  const double dx = __dsub_rn(q.x, p.x), dy = __dsub_rn(q.y, p.y);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// CWvertexEdge (R1: sweep_out(x) = next(twin(x))): next of an interior half-edge is
// next_in, of a border half-edge the exterior chain
__device__ __forceinline__ int32_t cw_vertex_edge(int32_t x, int64_t T3, const int32_t* __restrict__ twin,
                                                  const int32_t* __restrict__ next) {
  const int32_t t = twin[x];
  return t >= T3 ? next[t] : next_in(t);
}

__device__ __forceinline__ bool fbit(const uint32_t* F, int64_t T3, int32_t x) { return x >= T3 || bit_of(F, x); }

// Alg. 7 (LLK): one thread per triangle: d1, d2, d3 = squared lengths of 3f, 3f+1, 3f+2
// (FP64, no FMA, R11); the first maximum (R7) is marked in the longest-edge bit-vector
__global__ void k_p_llk(int64_t T, const double2* __restrict__ xy, const int32_t* __restrict__ origin, uint32_t* Lb,
                        const DevCounters* ctr) {
  if (ctr->status) return;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < T; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = origin[3 * f], b = origin[3 * f + 1], c = origin[3 * f + 2];
    const double d0 = sq_len_p(xy, a, b), d1 = sq_len_p(xy, b, c), d2 = sq_len_p(xy, c, a);
    int k = 0;
    double dk = d0;
    if (d1 > dk) { k = 1; dk = d1; }
    if (d2 > dk) k = 2;
    const int64_t e = 3 * f + k;
    atomicOr(&Lb[e >> 5], 1u << (e & 31));
  }
}

// Alg. 8 (LFK) and Alg. 9 (LSK): one thread per interior half-edge; a warp owns 32
// consecutive half-edges = one bit-vector word
__global__ void k_p_lfk(int64_t T, const int32_t* __restrict__ twin, const uint32_t* __restrict__ Lb, uint32_t* F0,
                        const DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T, nw = (T3 + 31) / 32;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw; w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t e = 32 * w + (threadIdx.x & 31);
    bool f = false;
    if (e < T3) {
      const int32_t t = twin[e];
      f = t >= T3 || (!bit_of(Lb, (int32_t)e) && !bit_of(Lb, t));  // is_border_edge or is_not_longest_edge (R15)
    }
    const uint32_t word = __ballot_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0) F0[w] = word;
  }
}

__global__ void k_p_lsk(int64_t T, const int32_t* __restrict__ twin, const uint32_t* __restrict__ Lb, uint32_t* S,
                        const DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T, nw = (T3 + 31) / 32;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw; w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t e = 32 * w + (threadIdx.x & 31);
    bool s = false;
    if (e < T3) {
      const int32_t t = twin[e];
      const bool Le = bit_of(Lb, (int32_t)e);
      // terminal edge (both halves longest; the smaller interior id, R8) or terminal border edge
      s = Le && (t >= T3 || (bit_of(Lb, t) && e < t));
    }
    const uint32_t word = __ballot_sync(0xffffffffu, s);
    if ((threadIdx.x & 31) == 0) S[w] = word;
  }
}

// edgeOfVertex (Listing 1's vertex record): an interior half-edge
// leaving each vertex (any: LEK's count does not depend on where the rotation starts)
__global__ void k_p_incident(int64_t T, const int32_t* __restrict__ origin, int32_t* incident) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < 3 * T; e += (int64_t)gridDim.x * blockDim.x)
    incident[origin[e]] = (int32_t)e;
}

// Alg. 10 (LEK): one thread per vertex; F1 starts as a copy of F0 (snapshot, R6)
__global__ void k_p_lek(int64_t V, int64_t T, const int32_t* __restrict__ incident, const int32_t* __restrict__ twin,
                        const int32_t* __restrict__ next, const uint32_t* __restrict__ F0, uint32_t* F1, uint32_t* S,
                        DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T, H = T3 + ctr->n_border;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e0 = incident[v];
    if (e0 < 0) continue;  // a vertex of no triangle
    int32_t he = e0, nf = 0;
    int64_t deg = 0;
    do {  // count the frontier edges around v
      nf += fbit(F0, T3, he);
      ++deg;
      he = cw_vertex_edge(he, T3, twin, next);
      if (deg > H) { raise_status(ctr, ST_WALK); break; }
    } while (he != e0);
    if (nf != 1 || deg > H) continue;
    atomicAdd(&ctr->n_tips, 1);
    he = e0;
    while (!fbit(F0, T3, he)) he = cw_vertex_edge(he, T3, twin, next);  // the frontier edge
    for (int64_t k = 0; k < (deg - 1) / 2; ++k) he = cw_vertex_edge(he, T3, twin, next);  // middle edge (R5)
    const int32_t th = twin[he];
    atomicOr(&F1[he >> 5], 1u << (he & 31));
    atomicOr(&F1[th >> 5], 1u << (th & 31));
    atomicOr(&S[he >> 5], 1u << (he & 31));
    atomicOr(&S[th >> 5], 1u << (th & 31));
  }
}

// Alg. 11 (CaK): one thread per interior half-edge: a frontier half-edge gets the next
// frontier half-edge rotating CW about its target (from next_in) and the previous one
// rotating CCW about its origin (from prev_in, sweep_in(y) = prev(twin(y))); the others
// keep next_in / prev_in (R14)
__global__ void k_p_cak(int64_t T, const int32_t* __restrict__ twin, const uint32_t* __restrict__ F1,
                        int32_t* __restrict__ next, int32_t* __restrict__ prev, DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < T3; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ei = (int32_t)e;
    int32_t nx = next_in(ei), pv = prev_in(ei);
    if (bit_of(F1, ei)) {
      int64_t steps = 0;
      while (!fbit(F1, T3, nx)) {  // twin of a non-frontier half-edge is interior
        nx = next_in(twin[nx]);
        if (++steps > T3) { raise_status(ctr, ST_WALK); break; }
      }
      steps = 0;
      while (!fbit(F1, T3, pv)) {
        pv = prev_in(twin[pv]);
        if (++steps > T3) { raise_status(ctr, ST_WALK); break; }
      }
    }
    next[ei] = nx;
    prev[ei] = pv;
  }
}

// Alg. 12 (SFK): one thread per seed: rotate CW to a frontier half-edge, move the seed there (R13)
__global__ void k_p_sfk(int64_t T, const int32_t* __restrict__ twin, const uint32_t* __restrict__ F1, uint32_t* S,
                        int64_t n_words, DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t T3 = 3 * T;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += (int64_t)gridDim.x * blockDim.x) {
    for (uint32_t b = S[w]; b; b &= b - 1) {
      const int32_t s = (int32_t)(32 * w + __ffs(b) - 1);
      int32_t x = s;
      int64_t steps = 0;
      while (!fbit(F1, T3, x)) {
        x = next_in(twin[x]);
        if (++steps > T3 || x == s) { raise_status(ctr, ST_WALK); break; }
      }
      if (x != s) {  // only non-frontier bits are cleared, only frontier bits set: no conflicts
        atomicAnd(&S[s >> 5], ~(1u << (s & 31)));
        atomicOr(&S[x >> 5], 1u << (x & 31));
      }
    }
  }
}

// Overwrite seeds (OSK): one thread per seed: walk the polygon, its minimum id becomes
// its seed; the loop length goes with it for the compaction
__global__ void k_p_osk(int64_t T, const int32_t* __restrict__ next, uint32_t* S, uint32_t* C, uint8_t* len,
                        int32_t* wlen, int64_t n_words, DevCounters* ctr) {
  if (ctr->status) return;
  const int64_t H = 3 * T + ctr->n_border;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += (int64_t)gridDim.x * blockDim.x) {
    for (uint32_t b = S[w]; b; b &= b - 1) {
      const int32_t init = (int32_t)(32 * w + __ffs(b) - 1);
      int32_t mn = init, cur = next[init];
      int64_t n = 1;
      while (cur != init) {
        mn = min(mn, cur);
        cur = next[cur];
        if (++n > H) { raise_status(ctr, ST_WALK); return; }
      }
      if (mn != init) atomicAnd(&S[init >> 5], ~(1u << (init & 31)));
      atomicOr(&S[mn >> 5], 1u << (mn & 31));
      len[mn] = len_code(n);
      const uint32_t bit = 1u << (mn & 31);
      if (!(atomicOr(&C[mn >> 5], bit) & bit)) atomicAdd(&wlen[mn >> 5], (int32_t)n);
    }
  }
}

}  // namespace

int launch_canon_scan(Ctx* c, cudaStream_t s);  // generate.cu: "Scan and compact"

int launch_paper(Ctx* c, cudaStream_t s) {
  const int64_t T = c->T, V = c->V, nw = c->n_words;
  // (this ablation keeps int32 half-edge ids: polylla_label_generate_paper refuses
  // meshes with 3T + max_border > INT32_MAX, where both readings agree)
  int32_t* twin = reinterpret_cast<int32_t*>(c->twin);
  int32_t* next = reinterpret_cast<int32_t*>(c->next);
  const unsigned g = 148 * 8;
  uint32_t* Lb = c->TB;  // the longest-edge bit-vector (TB is unused on this path)
  int32_t* incident = reinterpret_cast<int32_t*>(c->vmap);  // dead after the build's border chaining
  int32_t* prev = reinterpret_cast<int32_t*>(c->left_key);  // CaK's prev (scratch: 24T B >= 4H)
  prof_mark(s, "p_LLK");
  cudaMemsetAsync(Lb, 0, (size_t)nw * 4, s);
  cudaMemsetAsync(c->C, 0, (size_t)nw * 4, s);  // (the build's in-tile canonical seeds are not used here)
  cudaMemsetAsync(c->wlen, 0, (size_t)nw * 4, s);
  k_p_llk<<<g, 256, 0, s>>>(T, reinterpret_cast<const double2*>(c->xy), c->origin, Lb, c->ctr);
  prof_mark(s, "p_LFK");
  k_p_lfk<<<g, 256, 0, s>>>(T, twin, Lb, c->F0, c->ctr);
  prof_mark(s, "p_LSK");
  k_p_lsk<<<g, 256, 0, s>>>(T, twin, Lb, c->S, c->ctr);
  prof_mark(s, "p_LEK");
  cudaMemsetAsync(incident, 0xFF, (size_t)V * 4, s);
  k_p_incident<<<g, 256, 0, s>>>(T, c->origin, incident);
  cudaMemcpyAsync(c->F1, c->F0, (size_t)nw * 4, cudaMemcpyDeviceToDevice, s);
  k_p_lek<<<g, 256, 0, s>>>(V, T, incident, twin, next, c->F0, c->F1, c->S, c->ctr);
  prof_mark(s, "p_CaK");
  k_p_cak<<<g, 256, 0, s>>>(T, twin, c->F1, next, prev, c->ctr);
  prof_mark(s, "p_SFK");
  k_p_sfk<<<g, 256, 0, s>>>(T, twin, c->F1, c->S, nw, c->ctr);
  prof_mark(s, "p_OSK");
  k_p_osk<<<g, 256, 0, s>>>(T, next, c->S, c->C, c->len, c->wlen, nw, c->ctr);
  prof_end(s);
  int n = 8;
  const int m = launch_canon_scan(c, s);
  if (m < 0) return -1;
  return cudaGetLastError() == cudaSuccess ? n + m : -1;
}

}  // namespace polylla
