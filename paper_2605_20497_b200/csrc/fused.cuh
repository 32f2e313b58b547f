// fused.cuh — pieces of the fused level-0 a2+a3 kernels shared by level0.cu (k_nbrscore, tier W)
// and hub.cu (key-partitioned hub nodes): the job, the Eq.6 validity test on one (key, acc)
// pair and the two top-Pi epilogues.
#pragma once
#include "score_common.cuh"

namespace hgp {

__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}


constexpr uint32_t kProbeCap = 64;   // longer probe runs mean the table is (nearly) full

struct FusedJob {
  ScoreJob S;                     // level arrays + parameters + cand
  const uint32_t *list, *list_count;   // nodes to process (nullptr: all of [lo, hi))
  uint32_t log2s;                 // table size
  uint32_t *pool;
  uint64_t pool_cap;
  unsigned long long *pool_cursor;
  uint64_t *start;                // [hi-lo] pool offset of each node's N(n)
  uint32_t *cnt;                  // [hi-lo]
  uint32_t *defer_list, *defer_count;     // table too small / wide -> next tier
  uint32_t *pool_list, *pool_count;       // pool full (cnt[n] holds the exact count) -> second pool
  uint64_t start_bias;                    // added to every start written
  const uint64_t *cv;                     // [E] c(e), Eq.5 term in 2^-24 fixed point
  const uint2 *wmu;                       // [N] (size, in_mu) packed for the validity test
  unsigned long long *tiers;              // work counters (hgp_tier_counts)
  int tier;
};

// Both epilogues write the node's best-first Pi list to crow[0..pi) (cand row, or a hub
// partition's partial row). Entry i of the node's (key, acc) list is dense[i]: a DenseSrc (the
// array the table sweep wrote) or a ListSrc (through the slot list, clearing the slot it reads).
struct DenseSrc {
  const uint2 *d;
  __device__ __forceinline__ uint2 operator[](uint32_t i) const { return d[i]; }
};
struct ListSrc {
  const uint16_t *slist;
  uint32_t keys_s, acc_s;   // shared-window addresses of keys[] / acc[]
  __device__ __forceinline__ uint2 operator[](uint32_t i) const {
    const uint32_t slot = slist[i];
    uint2 d;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d.x) : "r"(keys_s + 4 * slot));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d.y) : "r"(acc_s + 4 * slot));
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(keys_s + 4 * slot), "r"(0xFFFFFFFFu) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(acc_s + 4 * slot), "r"(0u) : "memory");
    return d;
  }
};
// The validity test of Eq.6 on one (key, acc) pair of the dense list; writes the
// N(n) entry (purge flag on invalid neighbours) and returns the shared-edge count and
// the neighbour. Every sum fits 32 bits: sizes sum to < 2^32 (reading #2), |in(n) ∪ in(m)| <= E.
struct EvalCtx {
  uint32_t wn, inn, imask, om32, de32, ib;
};
__device__ __forceinline__ EvalCtx eval_ctx(const ScoreJob &J, uint32_t n, uint32_t ib) {
  EvalCtx e;
  e.wn = J.node_w[n];
  e.inn = J.in_mu[n];
  e.ib = ib;
  e.imask = ib ? (uint32_t)((1ull << ib) - 1) : 0u;
  e.om32 = J.omega >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)J.omega;
  e.de32 = J.delta >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)J.delta;   // HGP_UNBOUNDED too
  return e;
}
__device__ __forceinline__ bool eval_one(const FusedJob &F, const EvalCtx &E, uint2 d, uint64_t pos, uint32_t &cnt) {
  const uint32_t v = d.x, x = d.y;
  cnt = E.ib < 32 ? x >> E.ib : 0u;
  const uint32_t inter = x & E.imask;
  const uint2 wm = __ldg(F.wmu + v);                               // (size(m), in_mu(m)): one gather
  // |in(n) ∪ in(m)| = in_mu(n) + in_mu(m) - inter; inter <= in_mu(m)
  const bool ok = E.wn + wm.x <= E.om32 && E.inn + (wm.y - inter) <= E.de32;
  F.pool[pos] = ok ? v : (v | kPurge);
  return ok;
}

// Phase 3 of k_nbrscore, PACKED: every score of the node is < 2^32 (S1 + cap < 2^32), so
// (score << 32 | id) is one u64 key ordering (score desc, id desc) exactly (Eq.6's max_id).
// Each warp takes chunks of 4 entries per lane; per chunk, pi rounds of a warp argmax (two 32-bit
// REDUX: the score word, then the id among its holders) over the chunk's keys and the warp's
// running list (carried by lanes 0..pi-1) rebuild that list. Warp 0 then merges the NW lists.
template <int PIMAX, int THREADS, class Src>
__device__ __forceinline__ void eval_packed(const ScoreJob &J, const FusedJob &F, uint32_t n, uint32_t count,
                                            const Src &dense, uint32_t g32, uint32_t ib, uint64_t base,
                                            uint64_t *s_tops, hgp_cand *crow) {
  constexpr uint32_t NW = THREADS / 32;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const EvalCtx E = eval_ctx(J, n, ib);
  const uint32_t cap32 = (uint32_t)J.noise_cap;
  uint64_t carry = 0;                                              // lane r < pi: the warp's r-th best
  for (uint32_t c0 = w * 32; c0 < count; c0 += 4 * THREADS) {     // warp-uniform
    uint64_t k[4];
    uint2 d[4], wm[4];
    // the 4 entries, then their 4 (size, in_mu) gathers in flight together, then the tests
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = c0 + u * THREADS + lane;
      d[u] = i < count ? dense[i] : make_uint2(kEmpty, 0u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) wm[u] = d[u].x != kEmpty ? __ldg(F.wmu + d[u].x) : make_uint2(0u, 0u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = c0 + u * THREADS + lane;
      k[u] = 0;
      if (d[u].x != kEmpty) {
        const uint32_t v = d[u].x, x = d[u].y;
        const uint32_t cnt = E.ib < 32 ? x >> E.ib : 0u;
        // |in(n) ∪ in(m)| = in_mu(n) + in_mu(m) - inter; inter <= in_mu(m)
        const bool ok = E.wn + wm[u].x <= E.om32 && E.inn + (wm[u].y - (x & E.imask)) <= E.de32;
        F.pool[base + i] = ok ? v : (v | kPurge);                  // purge flag
        if (ok) {
          uint32_t s32 = cnt * g32;                                // eta(n, m) < 2^32
          if (cap32) {
            const uint64_t key = ((uint64_t)min(n, v) << 32) | max(n, v);
            s32 += (uint32_t)__umul64hi(splitmix64(key ^ J.seed_mix), J.noise_cap + 1);   // uniform in [0, cap]
          }
          k[u] = ((uint64_t)s32 << 32) | v;
        }
      }
    }
    uint64_t nc = 0;
    for (uint32_t r = 0; r < J.pi; ++r) {
      uint64_t lm = carry;
#pragma unroll
      for (int u = 0; u < 4; ++u) lm = k[u] > lm ? k[u] : lm;
      const uint32_t hi = (uint32_t)(lm >> 32);
      const uint32_t mhi = __reduce_max_sync(0xFFFFFFFFu, hi);
      if (mhi == 0) break;                                         // every score >= 1: nothing left
      const uint32_t mlo = __reduce_max_sync(0xFFFFFFFFu, hi == mhi ? (uint32_t)lm : 0u);
      const uint64_t K = ((uint64_t)mhi << 32) | mlo;              // ids are distinct: one holder
      if (carry == K) carry = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k[u] == K) k[u] = 0;
      if (lane == r) nc = K;
    }
    carry = nc;
  }
  if (lane < J.pi) s_tops[w * PIMAX + lane] = carry;
  __syncthreads();
  if (w == 0) {
    TopK<PIMAX> t2;
#pragma unroll
    for (int i = 0; i < PIMAX; ++i) t2.k[i] = 0;
    for (uint32_t i = lane; i < NW * J.pi; i += 32) topk_insert<PIMAX>(t2, J.pi, s_tops[(i / J.pi) * PIMAX + i % J.pi]);
    warp_topk_merge<PIMAX>(t2, J.pi, s_tops + NW * PIMAX);
    __syncwarp();
    for (uint32_t r = lane; r < J.pi; r += 32) {
      const uint64_t kk = s_tops[NW * PIMAX + r];
      hgp_cand cd;
      cd.score = kk >> 32;
      cd.id = kk ? (uint32_t)kk : kNone;
      cd.pad = 0;
      crow[r] = cd;
    }
  }
}

// Phase 3, general: scores up to 2^62 as (u64 score, id) lists per thread, merged per warp and
// by warp 0.
template <int PIMAX, int THREADS, class Src>
__device__ __forceinline__ void eval_top(const ScoreJob &J, const FusedJob &F, uint32_t n, uint32_t count,
                                         const Src &dense, uint64_t g, uint32_t ib, uint64_t base, uint64_t *s_tops,
                                         uint32_t *s_topi, hgp_cand *crow) {
  constexpr uint32_t NW = THREADS / 32;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const EvalCtx E = eval_ctx(J, n, ib);
  Top<PIMAX> top;
#pragma unroll
  for (int i = 0; i < PIMAX; ++i) { top.s[i] = 0; top.id[i] = 0; }
  for (uint32_t i = tid; i < count; i += THREADS) {
    const uint2 d = dense[i];
    uint32_t cnt;
    if (!eval_one(F, E, d, base + i, cnt)) continue;
    uint64_t sc = (uint64_t)cnt * g;
    if (J.noise_cap) {
      const uint64_t key = ((uint64_t)min(n, d.x) << 32) | max(n, d.x);
      sc += __umul64hi(splitmix64(key ^ J.seed_mix), J.noise_cap + 1);
    }
    top_insert<PIMAX>(top, J.pi, sc, d.x);
  }
  warp_top_merge<PIMAX>(top, J.pi, s_tops + w * PIMAX, s_topi + w * PIMAX);
  __syncthreads();
  if (w == 0) {
    Top<PIMAX> t2;
#pragma unroll
    for (int i = 0; i < PIMAX; ++i) { t2.s[i] = 0; t2.id[i] = 0; }
    for (uint32_t i = lane; i < NW * J.pi; i += 32) {
      const uint32_t ww = i / J.pi, r = i % J.pi;
      top_insert<PIMAX>(t2, J.pi, s_tops[ww * PIMAX + r], s_topi[ww * PIMAX + r]);
    }
    warp_top_merge<PIMAX>(t2, J.pi, s_tops + NW * PIMAX, s_topi + NW * PIMAX);
    __syncwarp();
    for (uint32_t r = lane; r < J.pi; r += 32) {
      hgp_cand cd;
      cd.score = s_tops[NW * PIMAX + r];
      cd.id = cd.score ? s_topi[NW * PIMAX + r] : kNone;
      cd.pad = 0;
      crow[r] = cd;
    }
  }
}


// hub.cu: the key-partitioned tier for the listed nodes (device list + host bound of its count);
// the nodes it cannot finish are appended to lu / lu_count for the unfused path.
hgp_status hub_tier(hgp_ctx *c, const FusedJob &F, const uint32_t *list, const uint32_t *list_count, uint32_t hcount,
                    uint32_t *lu, uint32_t *lu_count);

}  // namespace hgp
