/* hgpgen — seeded synthetic directed-hypergraph generators (see hgpgen.h).
 * Inputs only: no step of the coarsening method lives here. */
#include "hgpgen.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- random numbers: splitmix64 seeding + xoshiro256** ---------------- */
typedef struct { uint64_t s[4]; } rng_t;

static uint64_t sm64(uint64_t *x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void rng_seed(rng_t *r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = sm64(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t rng_next(rng_t *r) {
  uint64_t *s = r->s;
  const uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
  s[2] ^= t; s[3] = rotl(s[3], 45);
  return res;
}
/* uniform integer in [0, n), Lemire's multiply-shift with rejection */
static inline uint64_t rng_below(rng_t *r, uint64_t n) {
  unsigned __int128 m = (unsigned __int128)rng_next(r) * n;
  uint64_t l = (uint64_t)m;
  if (l < n) {
    uint64_t t = (0 - n) % n;
    while (l < t) { m = (unsigned __int128)rng_next(r) * n; l = (uint64_t)m; }
  }
  return (uint64_t)(m >> 64);
}
static inline double rng_unit(rng_t *r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

/* ---------------- growable output ---------------- */
typedef struct {
  hgpgen_graph g;
  uint64_t cap;
} builder_t;

static int b_init(builder_t *b, uint32_t N, uint32_t E, uint64_t pin_cap) {
  memset(b, 0, sizeof(*b));
  b->g.num_nodes = N; b->g.num_edges = E;
  b->g.edge_off = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)E + 1));
  b->g.edge_nsrc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(E ? E : 1));
  b->g.edge_w = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(E ? E : 1));
  b->g.node_w = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(N ? N : 1));
  b->cap = pin_cap ? pin_cap : 16;
  b->g.pins = (uint32_t *)malloc(sizeof(uint32_t) * b->cap);
  if (!b->g.edge_off || !b->g.edge_nsrc || !b->g.edge_w || !b->g.node_w || !b->g.pins) return -1;
  b->g.edge_off[0] = 0;
  return 0;
}
static int b_reserve(builder_t *b, uint64_t extra) {
  if (b->g.num_pins + extra <= b->cap) return 0;
  uint64_t nc = b->cap * 2;
  while (nc < b->g.num_pins + extra) nc *= 2;
  uint32_t *p = (uint32_t *)realloc(b->g.pins, sizeof(uint32_t) * nc);
  if (!p) return -1;
  b->g.pins = p; b->cap = nc;
  return 0;
}

void hgpgen_free(hgpgen_graph *g) {
  if (!g) return;
  free(g->edge_off); free(g->edge_nsrc); free(g->pins); free(g->edge_w); free(g->node_w);
  memset(g, 0, sizeof(*g));
}

/* ---------------- C1 tiny ---------------- */
int hgpgen_tiny(uint64_t seed, uint32_t N, uint32_t E, uint32_t size_base, uint32_t size_binom,
                uint32_t in_cap, uint32_t wmax_e, uint32_t wmax_n, hgpgen_graph *out) {
  builder_t b;
  if (N < 2 || b_init(&b, N, E, (uint64_t)E * (size_base + size_binom / 2 + 1) + 16)) return -1;
  rng_t r; rng_seed(&r, seed);
  uint32_t *stamp = (uint32_t *)calloc(N, sizeof(uint32_t));   /* edge id + 1 that used node */
  uint32_t *indeg = (uint32_t *)calloc(N, sizeof(uint32_t));
  if (!stamp || !indeg) return -1;
  for (uint32_t n = 0; n < N; ++n) b.g.node_w[n] = wmax_n > 1 ? 1 + (uint32_t)rng_below(&r, wmax_n) : 1;
  for (uint32_t e = 0; e < E; ++e) {
    uint32_t sz = size_base;
    for (uint32_t i = 0; i < size_binom; ++i) sz += (uint32_t)(rng_next(&r) >> 63);
    if (sz > N) sz = N;
    if (sz < 1) sz = 1;
    double u = rng_unit(&r);
    uint32_t ns = u < 0.8 ? 1 : (u < 0.9 ? 0 : 2);
    if (ns > sz) ns = sz;
    b_reserve(&b, sz);
    uint32_t *dst = b.g.pins + b.g.num_pins;
    uint32_t got = 0;
    for (uint32_t i = 0; i < sz; ++i) {
      int is_dst = i >= ns;
      uint32_t n = 0; int ok = 0;
      for (int attempt = 0; attempt < 64 && !ok; ++attempt) {
        n = (uint32_t)rng_below(&r, N);
        ok = stamp[n] != e + 1 && (!is_dst || indeg[n] < in_cap);
      }
      if (!ok) continue;                       /* give up on this pin: edge gets smaller */
      stamp[n] = e + 1;
      if (is_dst) indeg[n]++;
      dst[got++] = n;
    }
    if (got == 0) {                            /* keep every edge non-empty: one source pin */
      uint32_t n = (uint32_t)rng_below(&r, N);
      dst[got++] = n; ns = 1;
    }
    if (ns > got) ns = got;
    b.g.num_pins += got;
    b.g.edge_off[e + 1] = b.g.num_pins;
    b.g.edge_nsrc[e] = ns;
    b.g.edge_w[e] = 1 + (uint32_t)rng_below(&r, wmax_e ? wmax_e : 1);
  }
  free(stamp); free(indeg);
  *out = b.g;
  return 0;
}

/* ---------------- C2/C5 SNN-mapping ---------------- */
int hgpgen_snn(uint64_t seed, uint32_t L, uint32_t R, uint32_t C, uint32_t F, uint32_t W,
               double rewire, hgpgen_graph *out) {
  uint64_t N64 = (uint64_t)L * R * C;
  if (N64 == 0 || N64 >= (1ull << 31) || W > R || W > C || F > W * W) return -1;
  uint32_t N = (uint32_t)N64, E = N;
  builder_t b;
  if (b_init(&b, N, E, (uint64_t)E * (F + 1))) return -1;
  rng_t r; rng_seed(&r, seed);
  uint32_t *win = (uint32_t *)malloc(sizeof(uint32_t) * W * W);
  uint32_t *stamp = (uint32_t *)calloc(N, sizeof(uint32_t));
  if (!win || !stamp) return -1;
  const uint32_t layer = R * C;
  for (uint32_t n = 0; n < N; ++n) {
    b.g.node_w[n] = 1;
    uint32_t l = n / layer, rc = n % layer, row = rc / C, col = rc % C;
    uint32_t tl = (l + 1) % L;
    int32_t r0 = (int32_t)row - (int32_t)(W / 2), c0 = (int32_t)col - (int32_t)(W / 2);
    if (r0 < 0) r0 = 0;
    if (c0 < 0) c0 = 0;
    if (r0 > (int32_t)(R - W)) r0 = (int32_t)(R - W);
    if (c0 > (int32_t)(C - W)) c0 = (int32_t)(C - W);
    uint32_t *seg = b.g.pins + b.g.num_pins;
    seg[0] = n;                                           /* the axon's source neuron */
    stamp[n] = n + 1;
    for (uint32_t i = 0; i < W * W; ++i) win[i] = i;
    for (uint32_t i = 0; i < F; ++i) {                    /* partial Fisher-Yates over the window */
      uint32_t j = i + (uint32_t)rng_below(&r, W * W - i);
      uint32_t t = win[i]; win[i] = win[j]; win[j] = t;
    }
    for (uint32_t i = 0; i < F; ++i) {                    /* window draws are distinct by construction */
      uint32_t wr = win[i] / W, wc = win[i] % W;
      seg[1 + i] = tl * layer + (uint32_t)(r0 + wr) * C + (uint32_t)(c0 + wc);
    }
    for (uint32_t i = 0; i < F; ++i) stamp[seg[1 + i]] = n + 1;
    if (rewire > 0) {
      for (uint32_t i = 0; i < F; ++i) {
        if (rng_unit(&r) >= rewire) continue;
        for (int attempt = 0; attempt < 64; ++attempt) {
          uint32_t m = tl * layer + (uint32_t)rng_below(&r, layer);
          if (stamp[m] == n + 1) continue;
          stamp[m] = n + 1;                               /* old pin's stamp stays: harmless */
          seg[1 + i] = m;
          break;
        }
      }
    }
    b.g.num_pins += F + 1;
    b.g.edge_off[n + 1] = b.g.num_pins;
    b.g.edge_nsrc[n] = 1;
    b.g.edge_w[n] = 1;
  }
  free(win); free(stamp);
  *out = b.g;
  return 0;
}

/* ---------------- C3/C4 VLSI-like ---------------- */
int hgpgen_vlsi(uint64_t seed, uint32_t N, uint32_t E, uint32_t dmin, uint32_t dmax, double alpha,
                double locality, uint32_t in_cap, hgpgen_graph *out) {
  if (N < 2 || dmin < 1 || dmax < dmin) return -1;
  if (dmax > N) dmax = N;
  if (dmin > dmax) dmin = dmax;
  builder_t b;
  if (b_init(&b, N, E, (uint64_t)E * 12 + 1024)) return -1;
  rng_t r; rng_seed(&r, seed);
  uint32_t K = dmax - dmin + 1;
  double *cdf = (double *)malloc(sizeof(double) * K);
  uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * N);
  uint32_t *stamp = (uint32_t *)calloc(N, sizeof(uint32_t));
  uint32_t *indeg = (uint32_t *)calloc(N, sizeof(uint32_t));
  if (!cdf || !perm || !stamp || !indeg) return -1;
  double acc = 0;
  for (uint32_t k = 0; k < K; ++k) { acc += pow((double)(dmin + k), -alpha); cdf[k] = acc; }
  for (uint32_t k = 0; k < K; ++k) cdf[k] /= acc;
  for (uint32_t i = 0; i < N; ++i) perm[i] = i;
  for (uint32_t i = N - 1; i > 0; --i) {
    uint32_t j = (uint32_t)rng_below(&r, (uint64_t)i + 1);
    uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  const double HN = log((double)N) + 0.5772156649015329;
  for (uint32_t n = 0; n < N; ++n) b.g.node_w[n] = 1;
  for (uint32_t e = 0; e < E; ++e) {
    double u = rng_unit(&r);
    uint32_t lo = 0, hi = K - 1;                             /* first k with cdf[k] >= u */
    while (lo < hi) { uint32_t mid = (lo + hi) / 2; if (cdf[mid] >= u) hi = mid; else lo = mid + 1; }
    uint32_t sz = dmin + lo;
    b_reserve(&b, sz);
    uint32_t *seg = b.g.pins + b.g.num_pins;
    uint32_t drv = (uint32_t)rng_below(&r, N);
    seg[0] = drv; stamp[drv] = e + 1;
    uint32_t got = 1;
    uint64_t half = 8ull * sz;
    uint64_t wlo = drv > half ? drv - half : 0, whi = (uint64_t)drv + half;
    if (whi > (uint64_t)N - 1) whi = N - 1;
    for (uint32_t i = 1; i < sz; ++i) {
      for (int attempt = 0; attempt < 64; ++attempt) {
        uint32_t m;
        if (rng_unit(&r) < locality) {
          m = (uint32_t)(wlo + rng_below(&r, whi - wlo + 1));
        } else {                                             /* Zipf(1) rank via inverse of H(k) ~ ln k + gamma */
          double t = rng_unit(&r) * HN - 0.5772156649015329;
          double kk = exp(t);
          uint64_t rank = kk < 1.0 ? 1 : (uint64_t)kk;
          if (rank > N) rank = N;
          m = perm[rank - 1];
        }
        if (stamp[m] == e + 1 || indeg[m] >= in_cap) continue;
        stamp[m] = e + 1; indeg[m]++;
        seg[got++] = m;
        break;
      }
    }
    b.g.num_pins += got;
    b.g.edge_off[e + 1] = b.g.num_pins;
    b.g.edge_nsrc[e] = 1;
    b.g.edge_w[e] = 1;
  }
  free(cdf); free(perm); free(stamp); free(indeg);
  *out = b.g;
  return 0;
}
