// radix.cu — stable LSD radix sort of (key, value) u32 pairs, CUB-free, single-pass ("onesweep")
// scatter per digit with decoupled look-back, and the incidence transpose built on it (a1).
//
// Incidence (reading #15): node n's list is in(n) ascending then out(n) ascending. With
// key(p) = pins[p] << 1 | [p is a src pin] and value(p) = edge(p) generated in pin order (edges
// ascending), a STABLE sort by key yields exactly that order: equal keys keep ascending edge
// ids, in-keys (…0) precede out-keys (…1). The sorted values are `inc`; inc_off / inc_nin are
// the key boundaries. No atomics decide any position, so the result is deterministic.
#include "csr_impl.cuh"
#include "lbs.cuh"
#include "scan.cuh"

namespace hgp {

constexpr int kRadixBits = 8, kRadixDigits = 1 << kRadixBits;
constexpr int kRsThreads = 512, kRsItems = 8, kRsWarps = kRsThreads / 32;
constexpr uint32_t kRsTile = kRsThreads * kRsItems;   // 4096 pairs per tile
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

// key / value generation from the edge CSR (pin order = ascending edge ids)
__global__ void __launch_bounds__(kLbsThreads) k_inc_keys(const uint64_t *edge_off, const uint32_t *edge_nsrc,
                                                          uint32_t E, uint64_t P, const uint32_t *pins,
                                                          uint32_t *keys, uint32_t *vals) {
  __shared__ LbsShared sh;
  const uint64_t p0 = (uint64_t)blockIdx.x * kLbsTile;
  lbs_stage(sh, edge_off, E, p0, P);
#pragma unroll 4
  for (int k = 0; k < kLbsItems; ++k) {
    const uint64_t p = p0 + (uint64_t)k * kLbsThreads + threadIdx.x;
    if (p >= P) break;
    const uint32_t e = lbs_edge(sh, edge_off, E, p);
    keys[p] = pins[p] << 1 | (p < edge_off[e] + edge_nsrc[e] ? 1u : 0u);
    vals[p] = e;
  }
}

// digit histograms of every pass at once: hist[pass][digit]
__global__ void __launch_bounds__(256) k_radix_hist(const uint32_t *keys, uint64_t n, uint32_t npass,
                                                    unsigned int *hist) {
  __shared__ unsigned int h[4][kRadixDigits];
  for (uint32_t i = threadIdx.x; i < 4 * kRadixDigits; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    for (uint32_t p = 0; p < npass; ++p) atomicAdd(&h[p][(k >> (p * kRadixBits)) & (kRadixDigits - 1)], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < npass * kRadixDigits; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(&hist[i], (&h[0][0])[i]);
}

// exclusive scan of each pass's 256 counts (one CTA of 256 threads)
__global__ void k_radix_bases(const unsigned int *hist, uint32_t npass, uint32_t *base) {
  __shared__ uint32_t w[8];
  for (uint32_t p = 0; p < npass; ++p) {
    const uint32_t v = hist[p * kRadixDigits + threadIdx.x];
    const uint32_t incl = warp_incl_scan(v);
    if ((threadIdx.x & 31) == 31) w[threadIdx.x >> 5] = incl;
    __syncthreads();
    uint32_t off = 0;
    for (uint32_t q = 0; q < (threadIdx.x >> 5); ++q) off += w[q];
    base[p * kRadixDigits + threadIdx.x] = off + incl - v;
    __syncthreads();
  }
}

// One stable scatter pass over digit (key >> shift) & 255. Tiles are claimed in order through an
// atomic counter, so every tile's predecessors are running or done (look-back cannot deadlock).
// Within a tile, element order is warp-major, then round, then lane — the input order — and the
// rank of an element among equal digits is counted in that order (match.any peers), so the pass
// is stable.
__global__ void __launch_bounds__(kRsThreads) k_radix_scatter(const uint32_t *keys, const uint32_t *vals,
                                                              uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                                                              uint32_t shift, const uint32_t *digit_base,
                                                              uint32_t *status, unsigned int *tile_ctr) {
  __shared__ uint32_t cnt[kRsWarps][kRadixDigits];   // per-warp digit counts, then per-warp offsets
  __shared__ uint32_t gbase[kRadixDigits];
  __shared__ uint32_t s_tile;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5, lt = (1u << lane) - 1;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (uint32_t i = tid; i < kRsWarps * kRadixDigits; i += kRsThreads) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * kRsTile + (uint64_t)w * (32 * kRsItems);
  uint32_t k[kRsItems], v[kRsItems], rk[kRsItems];
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const uint64_t i = t0 + (uint64_t)r * 32 + lane;
    k[r] = i < n ? keys[i] : 0u;
    v[r] = i < n ? vals[i] : 0u;
  }
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const uint64_t i = t0 + (uint64_t)r * 32 + lane;
    const uint32_t d = i < n ? (k[r] >> shift) & (kRadixDigits - 1) : kRadixDigits;   // tail: own class
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t before = d < kRadixDigits ? cnt[w][d] : 0u;
    rk[r] = before + __popc(peers & lt);
    __syncwarp();
    if (d < kRadixDigits && (peers & lt) == 0) cnt[w][d] = before + __popc(peers);   // the peers' leader
    __syncwarp();
  }
  __syncthreads();
  // per digit (one thread each): exclusive offsets over warps, tile total, look-back
  if (tid < kRadixDigits) {
    const uint32_t d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < kRsWarps; ++q) { const uint32_t x = cnt[q][d]; cnt[q][d] = run; run += x; }
    volatile uint32_t *st = status;
    if (tile == 0) {
      st[d] = kFlagInc | run;
      gbase[d] = digit_base[d];
    } else {
      st[(uint64_t)tile * kRadixDigits + d] = kFlagAgg | run;
      uint32_t prefix = 0;
      for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
        uint32_t x;
        do { x = st[(uint64_t)t * kRadixDigits + d]; } while ((x >> 30) == 0);
        prefix += x & kValMask;
        if ((x >> 30) == 2) break;
      }
      __threadfence();
      st[(uint64_t)tile * kRadixDigits + d] = kFlagInc | (prefix + run);
      gbase[d] = digit_base[d] + prefix;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const uint64_t i = t0 + (uint64_t)r * 32 + lane;
    if (i < n) {
      const uint32_t d = (k[r] >> shift) & (kRadixDigits - 1);
      const uint64_t dst = (uint64_t)gbase[d] + cnt[w][d] + rk[r];
      keys_out[dst] = k[r];
      vals_out[dst] = v[r];
    }
  }
}

// Stable sort of (keys, vals)[0, n) by key < 2^kbits. Sorted output ends in (*ko, *vo), which is
// either (keys, vals) or (keys_alt, vals_alt). n < 2^30.
hgp_status radix_sort_pairs(hgp_ctx *c, uint32_t *keys, uint32_t *vals, uint32_t *keys_alt, uint32_t *vals_alt,
                            uint64_t n, uint32_t kbits, uint32_t **ko, uint32_t **vo) {
  *ko = keys;
  *vo = vals;
  if (n <= 1) return HGP_OK;
  if (n >= (1ull << 30)) return set_error(HGP_E_OVERFLOW, "radix sort: more than 2^30 elements");
  const uint32_t npass = kbits ? (kbits + kRadixBits - 1) / kRadixBits : 1;
  if (npass > 4) return set_error(HGP_E_ARG, "radix sort: keys wider than 32 bits");
  const uint64_t tiles = (n + kRsTile - 1) / kRsTile;
  hgp_status st = HGP_OK;
  unsigned int *hist = scratch_zero<unsigned int>(c, 4 * kRadixDigits + 4, &st);
  uint32_t *base = scratch_raw<uint32_t>(c, 4 * kRadixDigits, &st);
  uint32_t *status = scratch_raw<uint32_t>(c, tiles * kRadixDigits, &st);
  if (st) return st;
  unsigned int *ctr = hist + 4 * kRadixDigits;
  const uint32_t gh = div_up(n, 256) < 4u * c->sm_count ? div_up(n, 256) : 4u * c->sm_count;
  HGP_TRY(launch(c, "radix_hist", k_radix_hist, dim3(gh), dim3(256), 0, (const uint32_t *)keys, n, npass, hist));
  HGP_TRY(launch(c, "radix_bases", k_radix_bases, dim3(1), dim3(kRadixDigits), 0, (const unsigned int *)hist, npass,
                 base));
  uint32_t *ks = keys, *vs = vals, *kd = keys_alt, *vd = vals_alt;
  for (uint32_t p = 0; p < npass; ++p) {
    HGP_CUDA(cudaMemsetAsync(status, 0, sizeof(uint32_t) * tiles * kRadixDigits, c->stream));
    HGP_CUDA(cudaMemsetAsync(ctr + p, 0, sizeof(unsigned int), c->stream));
    HGP_TRY(launch(c, "radix_scatter", k_radix_scatter, dim3((uint32_t)tiles), dim3(kRsThreads), 0,
                   (const uint32_t *)ks, (const uint32_t *)vs, kd, vd, n, p * kRadixBits,
                   (const uint32_t *)(base + p * kRadixDigits), status, ctr + p));
    uint32_t *tk = ks, *tv = vs;
    ks = kd; vs = vd; kd = tk; vd = tv;
  }
  *ko = ks;
  *vo = vs;
  return HGP_OK;
}

// inc_off[n] = first position of key 2n, inc_nin[n] = (first position of 2n+1) - inc_off[n]:
// every position i where the key changes fills the start of each key in (key[i-1], key[i]].
__global__ void k_inc_bounds(const uint32_t *skeys, uint64_t P, uint32_t N, uint64_t *inc_off, uint32_t *start1) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= P; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t kp = i == 0 ? 0 : (uint64_t)skeys[i - 1] + 1;     // first key not yet started
    const uint64_t kc = i == P ? 2ull * N : (uint64_t)skeys[i];      // keys kp..kc start at i
    for (uint64_t key = kp; key <= kc && key < 2ull * N + 1; ++key) {
      if (key == 2ull * N) { inc_off[N] = i; continue; }
      if (key & 1) start1[key >> 1] = (uint32_t)(i - 0);              // relative fix-up below
      else inc_off[key >> 1] = i;
    }
  }
}

// inc_nin = start1 - inc_off (start1 was stored as an absolute position truncated to u32 when
// P < 2^32, which the caller guarantees); in_mu = sum of mu over the in-list.
__global__ void k_inc_finish(const uint64_t *inc_off, const uint32_t *start1, const uint32_t *inc,
                             const uint32_t *edge_mu, uint32_t N, uint32_t *inc_nin, uint32_t *in_mu,
                             unsigned int *maxdeg) {
  const uint32_t lane = lane_id();
  uint32_t mx = 0;
  for (uint32_t n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += gridDim.x * (blockDim.x >> 5)) {
    const uint64_t a = inc_off[n], b = (uint64_t)start1[n];
    const uint32_t nin = (uint32_t)(b - a);
    uint32_t s = 0;
    for (uint64_t k = a + lane; k < b; k += 32) s += edge_mu[inc[k]];
    s = warp_sum(s);
    if (lane == 0) { inc_nin[n] = nin; in_mu[n] = s; }
    mx = max(mx, (uint32_t)(inc_off[n + 1] - a));
  }
  mx = warp_max(mx);
  if (lane == 0) atomicMax(maxdeg, mx);
}

// a1's transpose by the radix sort. Requires P < 2^30 (radix sort) and N < 2^31.
hgp_status build_incidence_radix(hgp_ctx *c, hgp_csr *g) {
  hgp_status st = HGP_OK;
  const uint32_t N = g->N, E = g->E;
  const uint64_t P = g->P;
  g->inc_off = dalloc_n<uint64_t>(c, (size_t)N + 1, &st);
  g->inc_nin = dalloc_n<uint32_t>(c, N, &st);
  g->inc = dalloc_n<uint32_t>(c, P, &st);
  g->in_mu = dalloc_n<uint32_t>(c, N, &st);
  uint32_t *k0 = scratch_raw<uint32_t>(c, P, &st);
  uint32_t *k1 = scratch_raw<uint32_t>(c, P, &st);
  uint32_t *v1 = scratch_raw<uint32_t>(c, P, &st);
  uint32_t *start1 = scratch_raw<uint32_t>(c, N ? N : 1, &st);
  unsigned int *d_max = scratch_zero<unsigned int>(c, 1, &st);
  if (st != HGP_OK) return st;
  // values are generated straight into g->inc so that an odd pass count ends there
  const uint32_t kbits = 33 - __builtin_clz((unsigned)(N ? N : 1));   // keys < 2N <= 2^kbits
  const uint32_t npass = (kbits + kRadixBits - 1) / kRadixBits;
  uint32_t *v0 = (npass & 1) && P > 1 ? v1 : g->inc;                // P <= 1: nothing to sort
  uint32_t *va = (npass & 1) ? g->inc : v1;
  HGP_TRY(launch(c, "inc_keys", k_inc_keys, dim3(div_up(P, kLbsTile)), dim3(kLbsThreads), 0,
                 (const uint64_t *)g->edge_off, (const uint32_t *)g->edge_nsrc, E, P, (const uint32_t *)g->pins, k0,
                 v0));
  uint32_t *ks = nullptr, *vs = nullptr;
  HGP_TRY(radix_sort_pairs(c, k0, v0, k1, va, P, kbits, &ks, &vs));
  if (vs != g->inc) return set_error(HGP_E_INTERNAL, "radix transpose: values not in place");
  const uint32_t gb = div_up(P + 1, 256) < 8u * c->sm_count ? div_up(P + 1, 256) : 8u * c->sm_count;
  HGP_TRY(launch(c, "inc_bounds", k_inc_bounds, dim3(gb), dim3(256), 0, (const uint32_t *)ks, P, N, g->inc_off,
                 start1));
  const uint32_t gf = N ? (div_up(N, 8) < 16u * c->sm_count ? div_up(N, 8) : 16u * c->sm_count) : 0;
  HGP_TRY(launch(c, "inc_finish", k_inc_finish, dim3(gf), dim3(256), 0, (const uint64_t *)g->inc_off,
                 (const uint32_t *)start1, (const uint32_t *)g->inc, (const uint32_t *)g->edge_mu, N, g->inc_nin,
                 g->in_mu, d_max));
  uint32_t mx = 0;
  HGP_TRY(read_back(c, d_max, 4, &mx));
  g->max_inc = mx;
  return HGP_OK;
}

}  // namespace hgp
