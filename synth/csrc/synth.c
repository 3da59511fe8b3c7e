/*
 * synth.c -- seeded synthetic triangulations (test + bench INPUT GENERATORS).
 *
 * This module is shared by both sides of the parity check (the CPU oracle in
 * oracle/ and the CUDA path in paper_2403_14723_b200/).  It holds none of the
 * Polylla method's arithmetic: no edge lengths, no labels, no half-edges.  It
 * only produces (xy, tri) inputs shaped like the paper's workloads:
 *
 *   - "Grid meshes":   Alg. 13, vertex k at (k div s, k mod s),
 *                      triangles (k,k+1,k+s+1),(k,k+s+1,k+s).  Loop bound fixed to
 *                      k < s*s - s (reading R10).  Optionally jittered:
 *                      interior vertices moved by a*(2u-1) per axis.
 *   - "Random meshes": uniform points in the unit square, points within delta of a
 *                      side snapped onto it, duplicates redrawn, Delaunay-triangulated
 *                      ("randomly placing points on a square, without
 *                      overlapping points ... tolerance parameter delta ... Delaunay").
 *                      The paper uses the Triangle tool; we use our own incremental
 *                      Lawson-flip Delaunay with EXACT integer predicates: points live
 *                      on the 2^24 x 2^24 lattice (x = u / 2^24 exactly in double), so
 *                      orient fits int64 and incircle fits __int128.
 *
 * Counter-based RNG (shared definition with synth/csrc/gridgen_dev.cu):
 *     synth_rng(seed, ctr) = splitmix64_mix(seed * 0x9E3779B97F4A7C15 + ctr + 1)
 *
 * Vertex ids are in RNG order (spatially random, like the Triangle input of the
 * paper); triangles are sorted by the Morton code of their lattice centroid,
 * vertex order within a triangle as produced (CCW).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define LAT_BITS 24
#define LAT_S ((int64_t)1 << LAT_BITS) /* lattice side: coordinates in [0, LAT_S] */

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t synth_rng(uint64_t seed, uint64_t ctr) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + ctr + 1ULL);
}
/* uniform double in [0,1) with 53 random bits */
static inline double rng_unit(uint64_t seed, uint64_t ctr) {
  return (double)(synth_rng(seed, ctr) >> 11) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------------- */
/* Alg. 13 grid (regular or jittered).  xy: [s*s][2], tri: [2(s-1)^2][3].      */
/* a == 0 gives the exact Alg. 13 integer grid.                               */
int64_t synth_grid(int64_t s, double a, uint64_t seed, double* xy, int32_t* tri) {
  if (s < 2) return -1;
  const int64_t n = s * s;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = k / s, j = k % s;
    double x = (double)i, y = (double)j;
    if (a != 0.0 && i > 0 && i < s - 1 && j > 0 && j < s - 1) {
      volatile double ux = rng_unit(seed, 2 * (uint64_t)k);
      volatile double uy = rng_unit(seed, 2 * (uint64_t)k + 1);
      volatile double tx = 2.0 * ux; tx = tx - 1.0; tx = a * tx; x = x + tx;
      volatile double ty = 2.0 * uy; ty = ty - 1.0; ty = a * ty; y = y + ty;
    }
    xy[2 * k] = x;
    xy[2 * k + 1] = y;
  }
  int64_t t = 0;
  for (int64_t k = 0; k < n - s; ++k) {
    if (k % s == s - 1) continue;
    tri[3 * t + 0] = (int32_t)k;
    tri[3 * t + 1] = (int32_t)(k + 1);
    tri[3 * t + 2] = (int32_t)(k + s + 1);
    ++t;
    tri[3 * t + 0] = (int32_t)k;
    tri[3 * t + 1] = (int32_t)(k + s + 1);
    tri[3 * t + 2] = (int32_t)(k + s);
    ++t;
  }
  return t;
}

/* ------------------------------------------------------------------------- */
/* random points on the lattice with border snapping and redraw of duplicates */

typedef struct { uint64_t* slot; uint64_t mask; } hset;
static int hset_insert(hset* h, uint64_t key) { /* key != 0; returns 1 if new */
  uint64_t i = mix64(key) & h->mask;
  for (;;) {
    if (h->slot[i] == 0) { h->slot[i] = key; return 1; }
    if (h->slot[i] == key) return 0;
    i = (i + 1) & h->mask;
  }
}

static inline uint64_t spread2(uint64_t v) { /* 32 bits -> even bits of 64 */
  v &= 0xFFFFFFFFULL;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFULL;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFULL;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0FULL;
  v = (v | (v << 2)) & 0x3333333333333333ULL;
  v = (v | (v << 1)) & 0x5555555555555555ULL;
  return v;
}
static inline uint64_t morton2(uint64_t x, uint64_t y) { return spread2(x) | (spread2(y) << 1); }

/* n points (n >= 4): ids 0..3 are the square's corners, ids 4.. are RNG draws.
 * delta_lat: snapping tolerance in lattice units.  px,py: lattice coordinates. */
static int gen_points(int64_t n, uint64_t seed, int64_t delta_lat, int32_t* px, int32_t* py) {
  uint64_t cap = 1;
  while (cap < (uint64_t)(2 * n + 16)) cap <<= 1;
  hset h = {(uint64_t*)calloc(cap, sizeof(uint64_t)), cap - 1};
  if (!h.slot) return -1;
  const int32_t cx[4] = {0, (int32_t)LAT_S, (int32_t)LAT_S, 0};
  const int32_t cy[4] = {0, 0, (int32_t)LAT_S, (int32_t)LAT_S};
  for (int c = 0; c < 4; ++c) {
    px[c] = cx[c]; py[c] = cy[c];
    hset_insert(&h, (((uint64_t)cx[c] << 32) | (uint64_t)cy[c]) + 1);
  }
  uint64_t ctr = 0;
  for (int64_t i = 4; i < n; ++i) {
    for (;;) {
      uint64_t r = synth_rng(seed, ctr++);
      int64_t x = (int64_t)(r >> 40);               /* 24 bits */
      int64_t y = (int64_t)((r >> 16) & 0xFFFFFF);  /* 24 bits */
      if (x < delta_lat) x = 0; else if (x > LAT_S - delta_lat) x = LAT_S;
      if (y < delta_lat) y = 0; else if (y > LAT_S - delta_lat) y = LAT_S;
      if (hset_insert(&h, (((uint64_t)x << 32) | (uint64_t)y) + 1)) {
        px[i] = (int32_t)x; py[i] = (int32_t)y;
        break;
      }
    }
  }
  free(h.slot);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* incremental Delaunay (Lawson flips), exact integer predicates              */

typedef struct {
  const int32_t* px; const int32_t* py;
  int32_t* tv;   /* [3*cap] vertex ids, CCW */
  int32_t* tn;   /* [3*cap] neighbour opposite vertex slot, -1 = hull */
  int64_t nt, cap;
  int32_t* stack; int64_t sp, scap;
} dt;

static inline int64_t orient(const dt* d, int32_t a, int32_t b, int32_t c) {
  const int64_t ax = d->px[a], ay = d->py[a];
  return (d->px[b] - ax) * (d->py[c] - ay) - (d->py[b] - ay) * (d->px[c] - ax);
}
static inline int incircle_pos(const dt* d, int32_t a, int32_t b, int32_t c, int32_t q) {
  const int64_t qx = d->px[q], qy = d->py[q];
  const int64_t adx = d->px[a] - qx, ady = d->py[a] - qy;
  const int64_t bdx = d->px[b] - qx, bdy = d->py[b] - qy;
  const int64_t cdx = d->px[c] - qx, cdy = d->py[c] - qy;
  const __int128 al = (__int128)(adx * adx + ady * ady);
  const __int128 bl = (__int128)(bdx * bdx + bdy * bdy);
  const __int128 cl = (__int128)(cdx * cdx + cdy * cdy);
  const __int128 det = al * (__int128)(bdx * cdy - cdx * bdy) +
                       bl * (__int128)(cdx * ady - adx * cdy) +
                       cl * (__int128)(adx * bdy - bdx * ady);
  return det > 0;
}

#define TV(t, i) d->tv[3 * (t) + (i)]
#define TN(t, i) d->tn[3 * (t) + (i)]

static inline void set_tri(dt* d, int64_t t, int32_t a, int32_t b, int32_t c, int32_t na, int32_t nb, int32_t nc) {
  TV(t, 0) = a; TV(t, 1) = b; TV(t, 2) = c;
  TN(t, 0) = na; TN(t, 1) = nb; TN(t, 2) = nc;
}
static inline void repoint(dt* d, int32_t nbr, int32_t from, int32_t to) {
  if (nbr < 0) return;
  for (int i = 0; i < 3; ++i)
    if (TN(nbr, i) == from) { TN(nbr, i) = to; return; }
}
static inline int push(dt* d, int32_t t) {
  if (d->sp >= d->scap) {
    d->scap *= 2;
    int32_t* s = (int32_t*)realloc(d->stack, (size_t)d->scap * sizeof(int32_t));
    if (!s) return -1;
    d->stack = s;
  }
  d->stack[d->sp++] = t;
  return 0;
}

/* legalize edges opposite p (p sits at vertex slot 0 of every pushed triangle) */
static int legalize(dt* d) {
  while (d->sp > 0) {
    const int32_t t = d->stack[--d->sp];
    const int32_t p = TV(t, 0), a = TV(t, 1), b = TV(t, 2);
    const int32_t u = TN(t, 0);
    if (u < 0) continue;
    int k = 0;
    while (TN(u, k) != t) ++k;
    const int32_t q = TV(u, k);
    if (!incircle_pos(d, p, a, b, q)) continue;
    const int32_t Nta = TN(t, 1), Ntb = TN(t, 2);
    const int32_t Nub = TN(u, (k + 1) % 3), Nua = TN(u, (k + 2) % 3);
    set_tri(d, t, p, a, q, Nub, u, Ntb);
    set_tri(d, u, p, q, b, Nua, Nta, t);
    repoint(d, Nub, u, t);
    repoint(d, Nta, t, u);
    if (push(d, t) || push(d, u)) return -1;
  }
  return 0;
}

static int insert_point(dt* d, int32_t p, int32_t* last, uint32_t* rs) {
  int32_t t = *last, prev = -1;
  int64_t steps = 0;
  for (;;) {
    if (++steps > 4 * d->nt + 16) return -2; /* walk failed */
    *rs ^= *rs << 13; *rs ^= *rs >> 17; *rs ^= *rs << 5;
    const int r = (int)(*rs % 3);
    int moved = 0;
    for (int ii = 0; ii < 3; ++ii) {
      const int i = (ii + r) % 3;
      const int32_t nb = TN(t, i);
      if (nb == prev && nb >= 0) continue;
      if (orient(d, TV(t, (i + 1) % 3), TV(t, (i + 2) % 3), p) < 0) {
        if (nb < 0) return -3; /* outside the square: impossible */
        prev = t; t = nb; moved = 1;
        break;
      }
    }
    if (moved) continue;
    /* all non-skipped edges are non-negative; check the skipped one too */
    int64_t o[3];
    int neg = 0;
    for (int i = 0; i < 3; ++i) {
      o[i] = orient(d, TV(t, (i + 1) % 3), TV(t, (i + 2) % 3), p);
      if (o[i] < 0) neg = 1;
    }
    if (neg) { prev = -1; continue; }
    int nz = 0, zi = -1;
    for (int i = 0; i < 3; ++i) if (o[i] == 0) { ++nz; zi = i; }
    if (nz >= 2) return -4; /* duplicate point */
    if (d->nt + 2 > d->cap) return -5;
    if (nz == 0) {
      const int32_t a = TV(t, 0), b = TV(t, 1), c = TV(t, 2);
      const int32_t n0 = TN(t, 0), n1 = TN(t, 1), n2 = TN(t, 2);
      const int32_t t0 = t, t1 = (int32_t)d->nt, t2 = (int32_t)d->nt + 1;
      d->nt += 2;
      set_tri(d, t0, p, b, c, n0, t1, t2);
      set_tri(d, t1, p, c, a, n1, t2, t0);
      set_tri(d, t2, p, a, b, n2, t0, t1);
      repoint(d, n1, t, t1);
      repoint(d, n2, t, t2);
      if (push(d, t0) || push(d, t1) || push(d, t2)) return -1;
    } else {
      const int i = zi;
      const int32_t a = TV(t, i), b = TV(t, (i + 1) % 3), c = TV(t, (i + 2) % 3);
      const int32_t na = TN(t, i), nb = TN(t, (i + 1) % 3), nc = TN(t, (i + 2) % 3);
      if (na < 0) {
        const int32_t t0 = t, t1 = (int32_t)d->nt;
        d->nt += 1;
        set_tri(d, t0, p, c, a, nb, t1, -1);
        set_tri(d, t1, p, a, b, nc, -1, t0);
        repoint(d, nc, t, t1);
        if (push(d, t0) || push(d, t1)) return -1;
      } else {
        const int32_t u = na;
        int k = 0;
        while (TN(u, k) != t) ++k;
        const int32_t q = TV(u, k);
        const int32_t mc = TN(u, (k + 1) % 3), mb = TN(u, (k + 2) % 3);
        const int32_t t0 = t, t1 = (int32_t)d->nt, u0 = u, u1 = (int32_t)d->nt + 1;
        d->nt += 2;
        set_tri(d, t0, p, c, a, nb, t1, u1);
        set_tri(d, t1, p, a, b, nc, u0, t0);
        set_tri(d, u0, p, b, q, mc, u1, t1);
        set_tri(d, u1, p, q, c, mb, t0, u0);
        repoint(d, nc, t, t1);
        repoint(d, mb, u, u1);
        if (push(d, t0) || push(d, t1) || push(d, u0) || push(d, u1)) return -1;
      }
    }
    *last = t;
    return legalize(d);
  }
}

typedef struct { uint64_t key; int64_t idx; } kv;
static int kv_cmp(const void* A, const void* B) {
  const kv* a = (const kv*)A; const kv* b = (const kv*)B;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* Random-point Delaunay mesh of the unit square.
 *   n:        number of vertices (>= 4), ids 0..3 = corners
 *   delta:    snapping tolerance (fraction of the side), e.g. 1/sqrt(n)
 *   xy:       out [n][2] doubles (exact lattice values / 2^24)
 *   tri:      out [tri_cap][3]
 * returns the triangle count T (= 2n - 2 - (#border vertices)... any), or < 0 on error. */
int64_t synth_random_delaunay(int64_t n, uint64_t seed, double delta, double* xy,
                              int32_t* tri, int64_t tri_cap) {
  if (n < 4) return -1;
  int32_t* px = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int32_t* py = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  if (!px || !py) return -1;
  const int64_t delta_lat = (int64_t)llround(delta * (double)LAT_S);
  if (gen_points(n, seed, delta_lat, px, py)) return -1;

  /* insertion order: Morton order of lattice coordinates */
  kv* ord = (kv*)malloc((size_t)n * sizeof(kv));
  for (int64_t i = 0; i < n; ++i) ord[i].key = morton2((uint64_t)px[i], (uint64_t)py[i]), ord[i].idx = i;
  qsort(ord + 4, (size_t)(n - 4), sizeof(kv), kv_cmp);

  dt D;
  dt* d = &D;
  d->px = px; d->py = py;
  d->cap = 2 * n + 8;
  d->tv = (int32_t*)malloc((size_t)d->cap * 3 * sizeof(int32_t));
  d->tn = (int32_t*)malloc((size_t)d->cap * 3 * sizeof(int32_t));
  d->scap = 1024;
  d->stack = (int32_t*)malloc((size_t)d->scap * sizeof(int32_t));
  d->sp = 0;
  if (!d->tv || !d->tn || !d->stack) return -1;
  /* initial square: corners 0=(0,0) 1=(S,0) 2=(S,S) 3=(0,S); tris (0,1,2),(0,2,3) */
  set_tri(d, 0, 0, 1, 2, -1, 1, -1);
  set_tri(d, 1, 0, 2, 3, -1, -1, 0);
  d->nt = 2;
  int32_t last = 0;
  uint32_t rs = 2463534242u;
  int64_t rc = 0;
  for (int64_t i = 4; i < n; ++i) {
    rc = insert_point(d, (int32_t)ord[i].idx, &last, &rs);
    if (rc) break;
  }
  int64_t T = d->nt;
  if (!rc && T > tri_cap) rc = -6;
  if (!rc) {
    /* sort triangles by Morton code of the lattice centroid (sum of 3 vertices) */
    kv* tk = (kv*)malloc((size_t)T * sizeof(kv));
    for (int64_t t = 0; t < T; ++t) {
      const uint64_t sx = (uint64_t)px[TV(t, 0)] + px[TV(t, 1)] + px[TV(t, 2)];
      const uint64_t sy = (uint64_t)py[TV(t, 0)] + py[TV(t, 1)] + py[TV(t, 2)];
      tk[t].key = morton2(sx, sy);
      tk[t].idx = t;
    }
    qsort(tk, (size_t)T, sizeof(kv), kv_cmp);
    for (int64_t t = 0; t < T; ++t) {
      const int64_t s = tk[t].idx;
      tri[3 * t + 0] = TV(s, 0);
      tri[3 * t + 1] = TV(s, 1);
      tri[3 * t + 2] = TV(s, 2);
    }
    free(tk);
    const double inv = 1.0 / (double)LAT_S;
    for (int64_t i = 0; i < n; ++i) {
      xy[2 * i] = (double)px[i] * inv;
      xy[2 * i + 1] = (double)py[i] * inv;
    }
  }
  free(ord); free(px); free(py); free(d->tv); free(d->tn); free(d->stack);
  return rc ? rc : T;
}

/* Random-point Delaunay in lattice units (int32) -- for exact-geometry tests. */
int64_t synth_random_points_lattice(int64_t n, uint64_t seed, double delta, int32_t* px, int32_t* py) {
  const int64_t delta_lat = (int64_t)llround(delta * (double)LAT_S);
  return gen_points(n, seed, delta_lat, px, py);
}
