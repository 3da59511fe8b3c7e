/*
 * polylla_oracle.c -- the sequential CPU Polylla ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2403_14723_b200) never links, imports or calls it, and this file shares no
 * code, header, table or helper with the CUDA path.
 *
 * It is a plain, slow, obviously-correct transcription of the paper's sequential
 * algorithm (Sec. 5, Alg. 1-6) over the half-edge structure of
 * Sec. 4 (L203-303), with the readings R1-R18 listed in DESIGN.md where the paper is
 * silent or garbled.  Every function cites the passage it follows.  Arithmetic on
 * coordinates is IEEE double with no FMA contraction (built with -ffp-contract=off,
 * reading R11).
 *
 * Conventions ("each three half-edges ... represent a face";
 * SPEC.md L39-40, L101):
 *   interior half-edge e = 3f + k, origin = tri'[f][k], target = tri'[f][(k+1)%3]
 *   next_in(e) = 3f + (k+1)%3, prev_in(e) = 3f + (k+2)%3
 *   border half-edges are numbered 3T + rank(e) over the unmatched interior e in
 *   ascending order (R9); the border half-edges chain around the exterior face.
 *
 * Parity pins: see tests/test_oracle_*.py (hand-worked fixtures, brute-force Lepp
 * regions, closed forms for grids, invariants).  No function here is unpinned.
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* status codes (same numeric meaning as include/polylla.h, defined independently) */
enum {
  OR_OK = 0,
  OR_E_INVALID_ARGUMENT = -1,
  OR_E_DANGLING_INDEX = -2,
  OR_E_DEGENERATE_TRI = -3,
  OR_E_NON_MANIFOLD_EDGE = -4,
  OR_E_NON_MANIFOLD_VERTEX = -5,
  OR_E_INDEX_OVERFLOW = -6,
  OR_E_WALK_BOUND = -8,
  OR_E_UNSEEDED_LOOP = -9,
  OR_E_NOMEM = -12
};

/* ---------------------------------------------------------------- half-edge mesh */
typedef struct {
  int64_t T, H, B, V;
  int64_t Hcap; /* capacity of origin/twin/next/prev (the build returns NOMEM if H exceeds it) */
  const double* xy;
  int32_t* origin; /* [H] */
  int32_t* twin;   /* [H] */
  int32_t* next;   /* [H] input-mesh next (triangles + exterior chain) */
  int32_t* prev;   /* [H] */
  int32_t* incident; /* [V] edgeOfVertex(v): smallest interior half-edge with origin v (Listing 1) */
} mesh;

static inline int is_border(const mesh* m, int64_t e) { return e >= 3 * m->T; }
static inline int64_t target(const mesh* m, int64_t e) { /* R2: target = origin(twin(e)) */
  return m->origin[m->twin[e]];
}
/* R1: rotation "by the edge it crosses": sweep_out(x) = next(twin(x)), the next
 * outgoing half-edge around origin(x) (the CWvertexEdge of Alg. 5, Fig. 7). */
static inline int64_t sweep_out(const mesh* m, int64_t x) { return m->next[m->twin[x]]; }

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct { uint64_t key; int64_t e; } edge_key;
static int edge_key_cmp(const void* A, const void* B) {
  const edge_key* a = (const edge_key*)A;
  const edge_key* b = (const edge_key*)B;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->e < b->e ? -1 : (a->e > b->e);
}

/* SPEC.md L45-53 build_from_triangles (realises PAPER.md L203-273):
 *  - dangling index -> DanglingIndex; zero signed area -> DegenerateTriangle;
 *  - CW triangles re-oriented by swapping v1,v2 (reading R10);
 *  - twins by grouping half-edges on the undirected key (min,max)
 *    -- here with a library sort; > 2 half-edges on a key, or two in the same
 *    direction -> NonManifoldEdge;
 *  - one border half-edge per unmatched interior half-edge (R9), chained around
 *    the boundary; a vertex with two outgoing border half-edges -> NonManifoldVertex.
 * Outputs origin/twin/next/prev of H = 3T + B half-edges. */
static int build(mesh* m, const int32_t* tri, int64_t* flips_out) {
  const int64_t T = m->T, V = m->V;
  const double* xy = m->xy;
  int64_t flips = 0;
  if (3 * T > INT32_MAX) return OR_E_INDEX_OVERFLOW;
  for (int64_t f = 0; f < T; ++f) {
    int32_t a = tri[3 * f], b = tri[3 * f + 1], c = tri[3 * f + 2];
    if (a < 0 || a >= V || b < 0 || b >= V || c < 0 || c >= V) return OR_E_DANGLING_INDEX;
    if (a == b || b == c || a == c) return OR_E_DEGENERATE_TRI;
    /* signed area (x_b-x_a)(y_c-y_a) - (y_b-y_a)(x_c-x_a), no FMA (R11) */
    const double area = (xy[2 * b] - xy[2 * a]) * (xy[2 * c + 1] - xy[2 * a + 1]) -
                        (xy[2 * b + 1] - xy[2 * a + 1]) * (xy[2 * c] - xy[2 * a]);
    if (area == 0.0) return OR_E_DEGENERATE_TRI;
    if (area < 0.0) { int32_t t = b; b = c; c = t; ++flips; }
    m->origin[3 * f] = a;
    m->origin[3 * f + 1] = b;
    m->origin[3 * f + 2] = c;
  }
  /* group interior half-edges by undirected key */
  edge_key* ek = (edge_key*)malloc((size_t)(3 * T) * sizeof(edge_key));
  if (!ek && T) return OR_E_NOMEM;
  for (int64_t e = 0; e < 3 * T; ++e) {
    const uint64_t o = (uint32_t)m->origin[e];
    const uint64_t t = (uint32_t)m->origin[3 * (e / 3) + (e % 3 + 1) % 3];
    const uint64_t lo = o < t ? o : t, hi = o < t ? t : o;
    ek[e].key = (lo << 32) | hi;
    ek[e].e = e;
  }
  qsort(ek, (size_t)(3 * T), sizeof(edge_key), edge_key_cmp);
  for (int64_t e = 0; e < 3 * T; ++e) m->twin[e] = -1;
  int rc = OR_OK;
  for (int64_t i = 0; i < 3 * T;) {
    int64_t j = i;
    while (j < 3 * T && ek[j].key == ek[i].key) ++j;
    if (j - i > 2) { rc = OR_E_NON_MANIFOLD_EDGE; break; }
    if (j - i == 2) {
      const int64_t e1 = ek[i].e, e2 = ek[i + 1].e;
      if (m->origin[e1] == m->origin[e2]) { rc = OR_E_NON_MANIFOLD_EDGE; break; }
      m->twin[e1] = (int32_t)e2;
      m->twin[e2] = (int32_t)e1;
    }
    i = j;
  }
  free(ek);
  if (rc) return rc;
  /* border half-edges: ids 3T + rank over unmatched interior e, ascending (R9) */
  int64_t B = 0;
  for (int64_t e = 0; e < 3 * T; ++e)
    if (m->twin[e] < 0) ++B;
  if (3 * T + B > INT32_MAX) return OR_E_INDEX_OVERFLOW;
  const int64_t H = 3 * T + B;
  if (H > m->Hcap) return OR_E_NOMEM;
  m->B = B;
  m->H = H;
  int64_t b = 3 * T;
  for (int64_t e = 0; e < 3 * T; ++e) {
    if (m->twin[e] >= 0) continue;
    m->twin[e] = (int32_t)b;
    m->twin[b] = (int32_t)e;
    m->origin[b] = m->origin[3 * (e / 3) + (e % 3 + 1) % 3]; /* origin(b) = target(e) */
    ++b;
  }
  /* interior next/prev: the triangle cycles */
  for (int64_t e = 0; e < 3 * T; ++e) {
    m->next[e] = (int32_t)(3 * (e / 3) + (e % 3 + 1) % 3);
    m->prev[e] = (int32_t)(3 * (e / 3) + (e % 3 + 2) % 3);
  }
  /* Vertex record's incident_halfedge, used by edgeOfVertex */
  if (m->incident) {
    for (int64_t v = 0; v < V; ++v) m->incident[v] = -1;
    for (int64_t e = 3 * T - 1; e >= 0; --e) m->incident[m->origin[e]] = (int32_t)e;
  }
  /* border chain: next(b) = the border half-edge whose origin is target(b) */
  int32_t* border_of = (int32_t*)malloc((size_t)(V ? V : 1) * sizeof(int32_t));
  if (!border_of) return OR_E_NOMEM;
  for (int64_t v = 0; v < V; ++v) border_of[v] = -1;
  for (int64_t x = 3 * T; x < H; ++x) {
    const int32_t v = m->origin[x];
    if (border_of[v] >= 0) { rc = OR_E_NON_MANIFOLD_VERTEX; break; }
    border_of[v] = (int32_t)x;
  }
  if (!rc) {
    for (int64_t x = 3 * T; x < H; ++x) {
      const int32_t nx = border_of[target(m, x)];
      if (nx < 0) { rc = OR_E_NON_MANIFOLD_VERTEX; break; }
      m->next[x] = nx;
      m->prev[nx] = (int32_t)x;
    }
  }
  free(border_of);
  *flips_out = flips;
  return rc;
}

/* Alg. 2 "CPU longest edge labeling": for each triangle t,
 * he = incidentHalfedge(t) = 3t; d1, d2, d3 = lengths of he, next(he), prev(he);
 * mark the max.  Squared lengths dx*dx + dy*dy with dx = x[target]-x[origin]
 * (SPEC.md L196); ties -> the first of (he, next, prev) attaining the max (R7).
 * Also returns the per-triangle code k* (0, 1, 2) for debugging/parity. */
static double sqlen(const mesh* m, int64_t e) {
  const int64_t o = m->origin[e], t = target(m, e);
  const double dx = m->xy[2 * t] - m->xy[2 * o];
  const double dy = m->xy[2 * t + 1] - m->xy[2 * o + 1];
  return dx * dx + dy * dy;
}
static void label_longest(const mesh* m, uint8_t* longest, uint8_t* lcode) {
  memset(longest, 0, (size_t)m->H);
  for (int64_t t = 0; t < m->T; ++t) {
    const int64_t he = 3 * t;
    const int64_t cand[3] = {he, m->next[he], m->prev[he]};
    const double d[3] = {sqlen(m, cand[0]), sqlen(m, cand[1]), sqlen(m, cand[2])};
    int best = 0;
    for (int k = 1; k < 3; ++k)
      if (d[k] > d[best]) best = k;
    longest[cand[best]] = 1;
    lcode[t] = (uint8_t)(cand[best] - he);
  }
}

/* Alg. 3 "Label frontier edges", with the condition read as
 * is_not_longest_edge? (R15): frontier[he] = (!L[he] && !L[twin he]) ||
 * border(he) || border(twin he). */
static void label_frontier(const mesh* m, const uint8_t* longest, uint8_t* frontier) {
  for (int64_t he = 0; he < m->H; ++he) {
    const int64_t tw = m->twin[he];
    const int is_not_longest = !longest[he] && !longest[tw];
    const int is_border_edge = is_border(m, he) || is_border(m, tw);
    frontier[he] = (uint8_t)(is_not_longest || is_border_edge);
  }
}

/* Alg. 4 "Label seed edges": terminal edge = both halves
 * longest and not border; terminal border edge = one half longest and border.
 * "Label he or twin(he) as seed" -> the interior half with the smaller id (R8).
 * Appends to the seed list in ascending order; returns its length. */
static int64_t label_seeds(const mesh* m, const uint8_t* longest, int32_t* seed_list) {
  int64_t n = 0;
  for (int64_t he = 0; he < m->H; ++he) {
    const int64_t tw = m->twin[he];
    const int border_edge = is_border(m, he) || is_border(m, tw);
    const int is_terminal_edge = longest[he] && longest[tw] && !border_edge;
    const int is_terminal_border_edge = (longest[he] || longest[tw]) && border_edge;
    if (!(is_terminal_edge || is_terminal_border_edge)) continue;
    int64_t rep;
    if (is_border(m, he)) rep = tw;
    else if (is_border(m, tw)) rep = he;
    else rep = he < tw ? he : tw;
    if (rep == he) seed_list[n++] = (int32_t)he;
  }
  return n;
}

/* Alg. 5 "Traversal phase: polygon construction", read per
 * R1/R3: rotate the seed with CWvertexEdge = sweep_out until frontier (init); then
 * repeatedly take in_curr = next(mesh_input[out_curr]) and rotate it with
 * sweep_out until frontier, set mesh_output[out].next = in, mesh_output[in].prev =
 * out, advance out_curr = in_curr, until back at init.  Returns init (the seed of
 * the generated polygon), or -1 when a walk exceeds H steps (InfiniteWalk). */
static int64_t traverse(const mesh* in, const uint8_t* frontier, int32_t* out_next,
                        int32_t* out_prev, int64_t seed) {
  int64_t he = seed, guard = 0;
  while (!frontier[he]) {
    he = sweep_out(in, he);
    if (++guard > in->H) return -1;
  }
  const int64_t init = he;
  int64_t out_curr = init;
  guard = 0;
  do {
    int64_t in_curr = in->next[out_curr];
    while (!frontier[in_curr]) {
      in_curr = sweep_out(in, in_curr);
      if (++guard > in->H) return -1;
    }
    out_next[out_curr] = (int32_t)in_curr;
    out_prev[in_curr] = (int32_t)out_curr;
    out_curr = in_curr;
    if (++guard > in->H) return -1;
  } while (out_curr != init);
  return init;
}

/* degree(v): number of outgoing half-edges met by rotating
 * around v from the outgoing half-edge e; -1 if no closure within H steps. */
static int64_t degree_from(const mesh* m, int64_t e) {
  int64_t x = e, d = 0;
  do {
    x = sweep_out(m, x);
    if (++d > m->H) return -1;
  } while (x != e);
  return d;
}

/* Barrier-tip test used by the repair phase: Alg. 10's criterion (PAPER.md
 * L717-723, "count frontier-edges adjacent to v ... equal to 1"), evaluated by a
 * full rotation around v starting at its outgoing half-edge e. */
static int64_t count_frontier_around(const mesh* m, const uint8_t* frontier, int64_t e) {
  int64_t x = e, c = 0, guard = 0;
  do {
    if (frontier[x]) ++c;
    x = sweep_out(m, x);
    if (++guard > m->H) return -1;
  } while (x != e);
  return c;
}

typedef struct {
  int64_t T, V;
  const double* xy;
  const int32_t* tri;
  /* outputs (caller-allocated, capacities: H <= 6T, P <= T, L <= 3T) */
  int32_t *origin, *twin, *next, *prev;
  int32_t* next_pre;     /* [H] mesh_output.next after the traversal phase (pre-repair) */
  uint8_t *lcode;        /* [T] */
  uint8_t *longest;      /* [H] */
  uint8_t *frontier0;    /* [H] after Alg. 3 */
  uint8_t *frontier1;    /* [H] after repair */
  int32_t *seeds0;       /* [<=H] seed list of Alg. 4 */
  int32_t *seeds;        /* [P] canonical seeds ascending */
  int32_t *offsets;      /* [P+1] */
  int32_t *loops;        /* [L] */
  int32_t *tips;         /* [<=V] barrier tips found (vertex ids, discovery order) */
  int64_t counts[10];    /* H, B, flips, n_seeds0, P, L, n_tips, n_mid_edges, rot_steps, 0 */
  double times[8];       /* Build, LM, LF, LS, Trav, Rep, Extract, total (seconds) */
  int64_t hcap;          /* capacity of the [H] arrays if > 0 (else 6T); memory only, not arithmetic */
} oracle_io;

/* Alg. 1: Label (Alg. 2-4) -> Traversal (Alg. 5 per seed) ->
 * Repair (Alg. 6 per polygon with barrier tips) -> polygons rebuilt from seeds
 * (PAPER.md L315), canonical seed = min half-edge id on the loop. */
int oracle_run(oracle_io* io) {
  const double t_start = now_s();
  const int64_t T = io->T;
  if (T < 1 || io->V < 3 || !io->xy || !io->tri) return OR_E_INVALID_ARGUMENT;
  /* mesh_input next/prev live in scratch; io->next/prev are mesh_output */
  const int64_t Hcap = io->hcap > 0 ? io->hcap : 6 * T;
  mesh M = {T, 0, 0, io->V, Hcap, io->xy, io->origin, io->twin, NULL, NULL, NULL};
  M.incident = (int32_t*)malloc((size_t)io->V * sizeof(int32_t));
  if (!M.incident) return OR_E_NOMEM;
  M.next = (int32_t*)malloc((size_t)Hcap * sizeof(int32_t));
  M.prev = (int32_t*)malloc((size_t)Hcap * sizeof(int32_t));
  if (!M.next || !M.prev) return OR_E_NOMEM;
  int64_t flips = 0;
  int rc = build(&M, io->tri, &flips);
  const double t_build = now_s();
  if (rc) { free(M.next); free(M.prev); free(M.incident); return rc; }
  const int64_t H = M.H;

  /* ---- Label phase */
  label_longest(&M, io->longest, io->lcode);
  const double t_lm = now_s();
  label_frontier(&M, io->longest, io->frontier0);
  const double t_lf = now_s();
  const int64_t n_seeds0 = label_seeds(&M, io->longest, io->seeds0);
  const double t_ls = now_s();

  /* ---- Traversal phase: mesh_output = copy of mesh_input */
  memcpy(io->next, M.next, (size_t)H * sizeof(int32_t));
  memcpy(io->prev, M.prev, (size_t)H * sizeof(int32_t));
  int64_t* poly_init = (int64_t*)malloc((size_t)(n_seeds0 + 1) * sizeof(int64_t));
  if (!poly_init) return OR_E_NOMEM;
  for (int64_t i = 0; i < n_seeds0; ++i) {
    poly_init[i] = traverse(&M, io->frontier0, io->next, io->prev, io->seeds0[i]);
    if (poly_init[i] < 0) { rc = OR_E_WALK_BOUND; break; }
  }
  memcpy(io->next_pre, io->next, (size_t)H * sizeof(int32_t));
  const double t_trav = now_s();

  /* ---- Repair phase (Alg. 6), per polygon with barrier tips.
   * Tips are taken on the unrepaired polygon with the Label-phase frontier F0
   * (snapshot, R6); the middle edge is floor((degree(b)-1)/2) CW rotations past
   * the frontier edge (R5); subseeds are re-traversed with the updated frontier. */
  memcpy(io->frontier1, io->frontier0, (size_t)H);
  int64_t n_final = 0, n_tips = 0, n_mid = 0;
  int64_t* final_init = (int64_t*)malloc((size_t)(n_seeds0 + 2 * io->V + 1) * sizeof(int64_t));
  int32_t* Lp = (int32_t*)malloc((size_t)(2 * io->V + 2) * sizeof(int32_t));
  uint8_t* A = (uint8_t*)calloc((size_t)H, 1);             /* usage bit-vector */
  uint8_t* tip_seen = (uint8_t*)calloc((size_t)io->V, 1);
  int64_t* poly_tips = (int64_t*)malloc((size_t)(io->V + 1) * sizeof(int64_t));
  if (!final_init || !Lp || !A || !tip_seen || !poly_tips) return OR_E_NOMEM;
  for (int64_t p = 0; p < n_seeds0 && !rc; ++p) {
    const int64_t init = poly_init[p];
    /* barrier tips of P: loop vertices with exactly one incident frontier edge */
    int64_t nt = 0, x = init;
    do {
      const int64_t v = M.origin[x];
      if (!tip_seen[v]) {
        const int64_t c = count_frontier_around(&M, io->frontier0, x);
        if (c < 0) { rc = OR_E_WALK_BOUND; break; }
        if (c == 1) { tip_seen[v] = 1; poly_tips[nt++] = v; }
      }
      x = io->next_pre[x];
    } while (x != init);
    if (rc) break;
    if (nt == 0) { final_init[n_final++] = init; continue; }
    int64_t nl = 0;
    for (int64_t i = 0; i < nt; ++i) {
      const int64_t b = poly_tips[i];
      int64_t e = M.incident[b]; /* line:searchfrontier: e = edgeOfVertex(b) */
      io->tips[n_tips++] = (int32_t)b;
      int64_t guard = 0;
      while (!io->frontier0[e]) { /* line:searchfrontier, on the snapshot F0 */
        e = sweep_out(&M, e);
        if (++guard > H) { rc = OR_E_WALK_BOUND; break; }
      }
      if (rc) break;
      const int64_t deg = degree_from(&M, e);
      if (deg < 0) { rc = OR_E_WALK_BOUND; break; }
      for (int64_t k = 0; k < (deg - 1) / 2; ++k) e = sweep_out(&M, e); /* line:midedge */
      io->frontier1[e] = 1;                                             /* line:labelmidedge */
      io->frontier1[M.twin[e]] = 1;
      Lp[nl++] = (int32_t)e;
      Lp[nl++] = M.twin[e];
      A[e] = 1;
      A[M.twin[e]] = 1;
      ++n_mid;
    }
    if (rc) break;
    for (int64_t i = 0; i < nl; ++i) {
      const int64_t h = Lp[i];
      if (!A[h]) continue;
      A[h] = 0;
      const int64_t pinit = traverse(&M, io->frontier1, io->next, io->prev, h);
      if (pinit < 0) { rc = OR_E_WALK_BOUND; break; }
      int64_t y = pinit;
      do { A[y] = 0; y = io->next[y]; } while (y != pinit);
      final_init[n_final++] = pinit;
    }
  }
  const double t_rep = now_s();

  /* ---- Output: one canonical seed per polygon (min half-edge id on the loop),
   * polygons ordered by it, CSR loops of origins. */
  int64_t P = 0, L = 0;
  if (!rc) {
    uint8_t* is_seed = (uint8_t*)calloc((size_t)H, 1);
    for (int64_t i = 0; i < n_final; ++i) {
      int64_t mn = final_init[i], y = final_init[i];
      do { if (y < mn) mn = y; y = io->next[y]; } while (y != final_init[i]);
      is_seed[mn] = 1;
    }
    for (int64_t e = 0; e < H; ++e) {
      if (!is_seed[e]) continue;
      io->seeds[P] = (int32_t)e;
      io->offsets[P] = (int32_t)L;
      int64_t y = e;
      do { io->loops[L++] = M.origin[y]; y = io->next[y]; } while (y != e);
      ++P;
    }
    io->offsets[P] = (int32_t)L;
    free(is_seed);
    /* every interior frontier half-edge on exactly one loop (R12) */
    int64_t nf = 0;
    for (int64_t e = 0; e < 3 * T; ++e) nf += io->frontier1[e];
    if (nf != L) rc = OR_E_UNSEEDED_LOOP;
  }
  const double t_ext = now_s();

  io->counts[0] = H; io->counts[1] = M.B; io->counts[2] = flips; io->counts[3] = n_seeds0;
  io->counts[4] = P; io->counts[5] = L; io->counts[6] = n_tips; io->counts[7] = n_mid;
  io->counts[8] = 0; io->counts[9] = 0;
  io->times[0] = t_build - t_start; io->times[1] = t_lm - t_build; io->times[2] = t_lf - t_lm;
  io->times[3] = t_ls - t_lf; io->times[4] = t_trav - t_ls; io->times[5] = t_rep - t_trav;
  io->times[6] = t_ext - t_rep; io->times[7] = t_ext - t_start;
  free(M.next); free(M.prev); free(M.incident); free(poly_init); free(final_init); free(Lp); free(A);
  free(tip_seen); free(poly_tips);
  return rc;
}

/* Stand-alone build for the mesh-core pins. */
int oracle_build(int64_t V, const double* xy, int64_t T, const int32_t* tri, int32_t* origin,
                 int32_t* twin, int32_t* next, int32_t* prev, int64_t* HB_flips) {
  mesh M = {T, 0, 0, V, 6 * T, xy, origin, twin, next, prev, NULL};
  int64_t flips = 0;
  const int rc = build(&M, tri, &flips);
  HB_flips[0] = M.H; HB_flips[1] = M.B; HB_flips[2] = flips;
  return rc;
}
