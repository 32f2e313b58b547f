// score_common.cuh — pieces shared by the a3 kernels (score.cu) and the fused level-0 a2+a3
// kernel (level0.cu): job description, top-Pi lists, gcd, Eq.5 edge term.
#pragma once
#include "common.cuh"

namespace hgp {

struct ScoreJob {
  // level
  const uint64_t *edge_off;
  const uint32_t *edge_nsrc, *pins, *edge_w, *edge_mu, *node_w;
  const uint64_t *inc_off;
  const uint32_t *inc_nin, *inc, *in_mu;
  // neighbours
  uint32_t lo, hi;
  const uint64_t *nb_off;      // CSR offsets relative to lo, or nullptr: segments nb_start/nb_len
  const uint64_t *nb_start;
  const uint32_t *nb_len;
  uint32_t *nbr;
  // params
  uint64_t omega, delta, noise_cap, seed_mix;
  uint32_t pi, norm;
  uint32_t E, N;               // edges / nodes of the level (per-edge and per-node precomputes)
  hgp_cand *cand;
  // scheduling
  const uint32_t *list;        // nodes of this launch (nullptr: every node of [lo,hi))
  const uint32_t *list_count;
  uint32_t cap;                // neighbour entries this tier holds (table load <= 1/2)
  uint32_t log2s;
  uint32_t *gtab;              // global tables when !SMEM
  uint32_t *big_list, *big_count;    // deferred: neighbourhood larger than cap
  uint32_t *wide_list, *wide_count;  // deferred: packed 32-bit accumulator would overflow
  const unsigned int *max_in_mu;     // device scalar: max in_mu over the level (nullptr: unknown)
  unsigned long long *tiers;         // work counters (hgp_tier_counts)
  int tier;
};

enum { kModeP32 = 0, kModeWide = 1, kModeSplit = 2 };

template <int PIMAX>
hgp_status launch_score_flat(hgp_ctx *c, ScoreJob J, uint32_t nn, uint32_t E, const uint64_t **cv_out = nullptr,
                             const uint2 **wmu_out = nullptr);
// score_hub.cu: the key-partitioned a3 tier for listed nodes with big N(n); the nodes it leaves
// are appended to lu / lu_count
template <int PIMAX>
hgp_status score_hub_t(hgp_ctx *c, const ScoreJob &J, const uint64_t *cv, const uint2 *wmu, const uint32_t *list,
                       const uint32_t *list_count, uint32_t hcount, uint32_t *lu, uint32_t *lu_count);

template <int PIMAX>
struct Top {   // best-first list of (score, id); empty entries are (0, 0): every real score >= 1
  uint64_t s[PIMAX];
  uint32_t id[PIMAX];
};

// (score desc, id desc): Eq.6's max_id argmax
__device__ __forceinline__ bool better(uint64_t s1, uint32_t i1, uint64_t s2, uint32_t i2) {
  return s1 > s2 || (s1 == s2 && i1 > i2);
}

template <int PIMAX>
__device__ __forceinline__ void top_insert(Top<PIMAX> &t, uint32_t pi, uint64_t s, uint32_t id) {
#pragma unroll
  for (int i = 0; i < PIMAX; ++i) {
    if (i < (int)pi && better(s, id, t.s[i], t.id[i])) {
      uint64_t ts = t.s[i]; uint32_t ti = t.id[i];
      t.s[i] = s; t.id[i] = id;
      s = ts; id = ti;
    }
  }
}

// pi rounds: warp argmax of the lanes' list heads; the winner lane pops its head. Lane 0 writes
// the merged best-first list to out_s/out_id[0..pi).
template <int PIMAX>
__device__ __forceinline__ void warp_top_merge(const Top<PIMAX> &top, uint32_t pi, uint64_t *out_s, uint32_t *out_id) {
  const uint32_t lane = lane_id();
  uint32_t head = 0;
  for (uint32_t r = 0; r < pi; ++r) {
    uint64_t hs = 0;
    uint32_t hid = 0;
#pragma unroll
    for (int i = 0; i < PIMAX; ++i)
      if (i == (int)head) { hs = top.s[i]; hid = top.id[i]; }
    uint32_t who = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t os = __shfl_xor_sync(0xFFFFFFFFu, hs, o);
      const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, hid, o);
      const uint32_t ow = __shfl_xor_sync(0xFFFFFFFFu, who, o);
      if (better(os, oi, hs, hid) || (os == hs && oi == hid && ow < who)) { hs = os; hid = oi; who = ow; }
    }
    if (lane == 0) { out_s[r] = hs; out_id[r] = hid; }
    if (hs != 0 && who == lane) ++head;
  }
}

// Packed keys (score << 32 | id) when every score of the node is < 2^32: one u64 compare orders
// (score desc, id desc) exactly. Empty entries are 0 (every real score >= 1).
template <int PIMAX>
struct TopK {
  uint64_t k[PIMAX];
};

template <int PIMAX>
__device__ __forceinline__ void topk_insert(TopK<PIMAX> &t, uint32_t pi, uint64_t key) {
#pragma unroll
  for (int i = 0; i < PIMAX; ++i) {
    if (i < (int)pi && key > t.k[i]) {
      const uint64_t x = t.k[i];
      t.k[i] = key;
      key = x;
    }
  }
}

// pi rounds of warp argmax over the lanes' list heads (keys are distinct unless empty).
template <int PIMAX>
__device__ __forceinline__ void warp_topk_merge(const TopK<PIMAX> &top, uint32_t pi, uint64_t *out) {
  const uint32_t lane = lane_id();
  uint32_t head = 0;
  for (uint32_t r = 0; r < pi; ++r) {
    uint64_t h = 0;
#pragma unroll
    for (int i = 0; i < PIMAX; ++i)
      if (i == (int)head) h = top.k[i];
    // u64 max as two 32-bit warp reductions (REDUX): the largest high word (score), then the
    // largest low word (id) among the lanes holding it
    const uint32_t hi = (uint32_t)(h >> 32);
    const uint32_t mhi = __reduce_max_sync(0xFFFFFFFFu, hi);
    const uint32_t mlo = __reduce_max_sync(0xFFFFFFFFu, hi == mhi ? (uint32_t)h : 0u);
    const uint64_t best = ((uint64_t)mhi << 32) | mlo;
    if (lane == 0) out[r] = best;
    if (best != 0 && h == best) ++head;
  }
}

__device__ __forceinline__ uint64_t gcd64(uint64_t a, uint64_t b) {
  if (a == 0) return b;
  if (b == 0) return a;
  const int sh = __ffsll((long long)(a | b)) - 1;
  a >>= __ffsll((long long)a) - 1;
  do {
    b >>= __ffsll((long long)b) - 1;
    if (a > b) { uint64_t t = a; a = b; b = t; }
    b -= a;
  } while (b);
  return a << sh;
}

__device__ __forceinline__ uint64_t edge_c(const ScoreJob &J, uint32_t e, uint64_t a, uint64_t b) {
  const uint64_t we = (uint64_t)J.edge_w[e] << HGP_FP_SHIFT;   // Eq.5 term, 2^-24 fixed point
  return J.norm ? we : we / (b - a);
}


__global__ void k_score_check(const uint32_t *node_w, const uint32_t *in_mu, uint32_t lo, uint32_t hi, uint64_t omega,
                              uint64_t delta, const uint64_t *edge_off, const uint32_t *edge_w, uint32_t E, uint32_t norm,
                              uint64_t *err, unsigned long long *wsum);
hgp_status score_prologue(hgp_ctx *c, const hgp_csr *g, uint32_t lo, uint32_t hi, const hgp_params *p, ScoreJob *J);
hgp_status score_finish(hgp_ctx *c);
hgp_status score_run(hgp_ctx *c, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p, hgp_cand *cand,
                     const uint32_t *list, const uint32_t *list_count);
// a3 for the nodes of a device list whose neighbours are segments start/len of nbr (relative
// to lo), with purge flags written in place; max_deg bounds the segment lengths.
hgp_status score_list_segments(hgp_ctx *c, ScoreJob J, uint32_t nn, uint32_t max_deg, const uint32_t *list,
                               const uint32_t *list_count);

}  // namespace hgp
