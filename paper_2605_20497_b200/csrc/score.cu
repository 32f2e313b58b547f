// score.cu — a3: candidate pairs proposal (§5.3; Eqs.5-6; top-Pi P:770).
//
// One CTA per node n. The unflagged entries of N(n) become the bins of an open-addressing
// table in shared memory (global memory for giant neighbourhoods); the CTA's warps walk
// the incident hyperedges (in-edges first) and their pins and accumulate, per bin,
//   eta(n,m)   += c(e)                     (Eq.5 in 2^-24 fixed point)
//   inter(n,m) += mu(e)  if e in in(n) and m in dst(e)
// with shared-memory atomics (integer sums: any order gives the same bits). Then every bin
// is validated (size(n)+size(m) <= Omega and in_mu(n)+in_mu(m)-inter <= Delta, Eq.6/P:623),
// invalid bins get the purge flag written back into N(n), and the top-Pi valid
// bins by (eta + noise desc, id desc) (Eq.6 max_id) become the candidates.
#include "csr_impl.cuh"
#include "hashset.cuh"
#include "score_common.cuh"

namespace hgp {

// One CTA per node. MODE kModeP32: one u32 per bin packs (eta/g) << ib | inter, where g is the
// gcd of the node's c(e) and ib = bits(in_mu(n)) (exact: inter <= in_mu(n) < 2^ib, and the
// node qualifies only if (sum c / g + 1) << ib <= 2^32); a single native shared-memory atomic
// add per pin visit. MODE kModeSplit (not launched: score_flat.cu's first tier runs split
// accumulators itself): u32 eta + u32 inter per bin (exact when sum c(e) over I(n)
// < 2^32: the usual case once hyperedge sizes differ and the gcd is 1); two native atomics per
// visit (the inter one only for dst pins of in-edges). MODE kModeWide: u64 eta (CAS loop) + u32
// inter per bin, for everything else.
template <int THREADS, int MODE, bool SMEM, int PIMAX>
__global__ void __launch_bounds__(THREADS) k_score(ScoreJob J) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint64_t s_tops[(THREADS / 32 + 1) * PIMAX];
  __shared__ uint32_t s_topi[(THREADS / 32 + 1) * PIMAX];
  __shared__ uint64_t s_sum[THREADS / 32], s_g[THREADS / 32];
  __shared__ uint32_t s_defer;
  __shared__ uint64_t s_gcd;
  __shared__ uint32_t s_ib;
  constexpr uint32_t NW = THREADS / 32;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t log2s = J.log2s, S = 1u << log2s;
  constexpr uint32_t SLOT = MODE == kModeP32 ? 8 : MODE == kModeSplit ? 12 : 16;
  unsigned char *base = SMEM ? dyn : reinterpret_cast<unsigned char *>(J.gtab) + ((size_t)blockIdx.x * SLOT << log2s);
  uint32_t *keys = reinterpret_cast<uint32_t *>(base);
  uint32_t *acc = reinterpret_cast<uint32_t *>(base + ((size_t)4 << log2s));        // P32 acc / wide inter
  uint64_t *eta = reinterpret_cast<uint64_t *>(base + ((size_t)8 << log2s));        // wide only
  uint32_t *inter32 = reinterpret_cast<uint32_t *>(base + ((size_t)8 << log2s) + 16);  // split only (S+1 slots)
  const uint32_t total = J.list_count ? *J.list_count : J.hi - J.lo;
  uint32_t done = 0;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t n = J.list ? J.list[t] : J.lo + t;
    uint64_t b0, b1;
    if (J.nb_off) { b0 = J.nb_off[n - J.lo]; b1 = J.nb_off[n - J.lo + 1]; }
    else { b0 = J.nb_start[n - J.lo]; b1 = b0 + J.nb_len[n - J.lo]; }
    if (b1 - b0 > J.cap) {                                        // larger tier (CTA-uniform)
      if (tid == 0) J.big_list[atomicAdd(J.big_count, 1u)] = n;
      continue;
    }
    // table of this node: the tier's shared table, or (global tables) just nextpow2(2 (|N(n)| + 1))
    // slots of the CTA's region, so clearing and probing cost what the node needs
    uint32_t nlog = log2s;
    if (!SMEM) {
      nlog = 6;
      while ((1ull << nlog) < 2 * (b1 - b0 + 1) + 2 && nlog < log2s) ++nlog;
    }
    const uint32_t Sn = 1u << nlog;
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    const uint32_t inn = J.in_mu[n];
    // ---- phase 0 (P32): gcd and sum of c(e) over I(n) decide whether the packed form is exact
    uint64_t g = 1;
    uint32_t ib = 0;
    if (MODE == kModeP32) {
      // S1 first; the gcd of c(e) (a binary-GCD reduction: thousands of instructions) only when
      // g = 1 leaves the packed form inexact
      uint64_t sum = 0;
      for (uint64_t k = i0 + tid; k < i1; k += THREADS) {
        const uint32_t e = J.inc[k];
        sum += edge_c(J, e, J.edge_off[e], J.edge_off[e + 1]);
      }
      sum = warp_sum(sum);
      if (lane == 0) s_sum[w] = sum;
      __syncthreads();
      uint64_t S1 = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) S1 += s_sum[q];
      const uint32_t bits = inn ? 32 - __clz(inn) : 0;
      if ((((unsigned __int128)(S1 + 1)) << bits) <= ((unsigned __int128)1 << 32)) {   // CTA-uniform
        g = 1;
        ib = bits;
        __syncthreads();                                          // s_sum is rewritten next node
      } else {
        uint64_t gg = 0;
        for (uint64_t k = i0 + tid; k < i1; k += THREADS) {
          const uint32_t e = J.inc[k];
          gg = gcd64(gg, edge_c(J, e, J.edge_off[e], J.edge_off[e + 1]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gg = gcd64(gg, __shfl_xor_sync(0xFFFFFFFFu, gg, o));
        if (lane == 0) s_g[w] = gg;
        __syncthreads();
        if (tid == 0) {
          uint64_t G1 = 0;
          for (uint32_t q = 0; q < NW; ++q) G1 = gcd64(G1, s_g[q]);
          if (G1 == 0) G1 = 1;
          const unsigned __int128 need = ((unsigned __int128)(S1 / G1 + 1)) << bits;
          s_defer = need > ((unsigned __int128)1 << 32);
          s_gcd = G1;
          s_ib = bits;
          if (s_defer) J.wide_list[atomicAdd(J.wide_count, 1u)] = n;
        }
        __syncthreads();
        if (s_defer) continue;                                    // CTA-uniform
        g = s_gcd;
        ib = s_ib;
      }
    }
    if (MODE == kModeSplit) {                                     // eta fits u32 iff sum c(e) < 2^32
      uint64_t sum = 0;
      for (uint64_t k = i0 + tid; k < i1; k += THREADS) {
        const uint32_t e = J.inc[k];
        sum += edge_c(J, e, J.edge_off[e], J.edge_off[e + 1]);
      }
      sum = warp_sum(sum);
      if (lane == 0) s_sum[w] = sum;
      __syncthreads();
      uint64_t S1 = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) S1 += s_sum[q];
      __syncthreads();                                            // s_sum is rewritten next node
      if (S1 >= (1ull << 32)) {                                   // CTA-uniform
        if (tid == 0) J.wide_list[atomicAdd(J.wide_count, 1u)] = n;
        continue;
      }
    }
    // ---- phase 1: bins = unflagged neighbours (+ n itself in P32 mode: every self-visit then
    // hits a real slot, no per-pin test; misses of purged neighbours go to a trash slot Sn)
    for (uint32_t i = tid; i < Sn; i += THREADS) {
      keys[i] = kEmpty;
      acc[i] = 0;
      if (MODE == kModeWide) eta[i] = 0;
      if (MODE == kModeSplit) inter32[i] = 0;
    }
    if (MODE != kModeWide && tid == 0) acc[Sn] = 0;
    if (MODE == kModeSplit && tid == 0) inter32[Sn] = 0;
    __syncthreads();
    for (uint64_t k = b0 + tid; k < b1; k += THREADS) {
      const uint32_t v = J.nbr[k];
      if (!(v & kPurge)) hs_insert(keys, nlog, v);
    }
    if (MODE != kModeWide && tid == 0) hs_insert(keys, nlog, n);
    __syncthreads();
    // ---- phase 2: traverse I(n): a warp loads the metadata of 32 incident edges at
    // once (lane = edge), then walks them; pins are fetched 128 at a time (4 per lane in flight).
    // Incident edges are dealt round-robin to warps (edge i0 + w + NW*l, l = 0, 1, ...): balanced.
    const uint32_t keys_s = opaque_u32(smem_u32addr(keys)), acc_s = opaque_u32(smem_u32addr(acc));
    const uint32_t inter_s = MODE == kModeSplit ? smem_u32addr(inter32) : 0u;
    const uint32_t hmask = Sn - 1;
    for (uint64_t kb = i0 + w; kb < i1; kb += (uint64_t)NW * 32) {
      const uint64_t k = kb + (uint64_t)NW * lane;
      uint64_t a = 0, ce = 0;
      uint32_t len = 0, srel = 0, mu_in = 0;
      if (k < i1) {
        const uint32_t e = J.inc[k];
        a = J.edge_off[e];
        const uint64_t b = J.edge_off[e + 1];
        len = (uint32_t)(b - a);
        srel = J.edge_nsrc[e];
        ce = edge_c(J, e, a, b);
        mu_in = k < iin ? J.edge_mu[e] : 0u;                       // e in in(n)
      }
      uint32_t add_s = 0, add_d = 0;
      if (MODE == kModeP32) {
        add_s = (uint32_t)((g == 1 ? ce : ce / g) << ib);
        add_d = add_s + mu_in;                                     // m in dst(e) and e in in(n)
      } else if (MODE == kModeSplit) {
        add_s = (uint32_t)ce;                                      // eta term
        add_d = mu_in;                                             // inter term of a dst pin
      }
      const uint32_t cnt = (uint32_t)min((uint64_t)32, (i1 - kb + NW - 1) / NW);
      for (uint32_t j = 0; j < cnt; ++j) {
        const uint64_t aj = __shfl_sync(0xFFFFFFFFu, a, j);
        const uint32_t lj = __shfl_sync(0xFFFFFFFFu, len, j);
        const uint32_t sj = __shfl_sync(0xFFFFFFFFu, srel, j);
        uint32_t as_j = 0, ad_j = 0, mu_j = 0;
        uint64_t ce_j = 0;
        if (MODE != kModeWide) {
          as_j = __shfl_sync(0xFFFFFFFFu, add_s, j);
          ad_j = __shfl_sync(0xFFFFFFFFu, add_d, j);
        } else {
          ce_j = __shfl_sync(0xFFFFFFFFu, ce, j);
          mu_j = __shfl_sync(0xFFFFFFFFu, mu_in, j);
        }
        const uint32_t *pj = J.pins + aj;
        for (uint32_t b4 = 0; b4 < lj; b4 += 128) {
          uint32_t m[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t idx = b4 + u * 32 + lane;
            m[u] = idx < lj ? __ldg(pj + idx) : kEmpty;
          }
          if constexpr (MODE != kModeWide) {
            // first probes of the 4 pins issued back to back (ILP), collisions resolved after
            uint32_t sl[4], kk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) sl[u] = hash_slot(m[u], nlog);
#pragma unroll
            for (int u = 0; u < 4; ++u) kk[u] = lds_u32(keys_s + 4 * sl[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (m[u] == kEmpty) continue;
              uint32_t slot = sl[u];
              if (kk[u] != m[u]) {
                uint32_t k2 = kk[u];
                while (true) {
                  if (k2 == kEmpty) { slot = Sn; break; }               // purged neighbour -> trash
                  slot = (slot + 1) & hmask;
                  k2 = lds_u32(keys_s + 4 * slot);
                  if (k2 == m[u]) break;
                }
              }
              const bool dst = b4 + u * 32 + lane >= sj;
              if constexpr (MODE == kModeP32) {
                red_add_u32(acc_s + 4 * slot, dst ? ad_j : as_j);
              } else {
                red_add_u32(acc_s + 4 * slot, as_j);
                if (dst && ad_j) red_add_u32(inter_s + 4 * slot, ad_j);
              }
            }
            continue;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (m[u] == kEmpty) continue;
            const bool dst = b4 + u * 32 + lane >= sj;
            {
              if (m[u] == n) continue;
              const uint32_t slot = hs_find(keys, nlog, m[u]);
              if (slot == kNone) continue;                          // purged neighbour
              atomicAdd(reinterpret_cast<unsigned long long *>(&eta[slot]), (unsigned long long)ce_j);
              if (dst && mu_j) atomicAdd(&acc[slot], mu_j);
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- phase 3: validity (Eq.6), purge flags, noise, per-thread top-pi
    Top<PIMAX> top;
#pragma unroll
    for (int i = 0; i < PIMAX; ++i) { top.s[i] = 0; top.id[i] = 0; }
    const uint64_t wn = J.node_w[n];
    const uint32_t imask = ib ? (uint32_t)((1ull << ib) - 1) : 0u;
    for (uint64_t k = b0 + tid; k < b1; k += THREADS) {
      const uint32_t v = J.nbr[k];
      if (v & kPurge) continue;
      const uint32_t slot = hs_find(keys, nlog, v);
      uint64_t e_nm, inter;
      if (MODE == kModeP32) {
        const uint32_t x = acc[slot];
        e_nm = (uint64_t)(ib < 32 ? x >> ib : 0) * g;
        inter = x & imask;
      } else if (MODE == kModeSplit) {
        e_nm = acc[slot];
        inter = inter32[slot];
      } else {
        e_nm = eta[slot];
        inter = acc[slot];
      }
      const uint64_t uni = (uint64_t)inn + J.in_mu[v] - inter;    // |in(n) ∪ in(m)|
      const bool ok = wn + J.node_w[v] <= J.omega && (J.delta == HGP_UNBOUNDED || uni <= J.delta);
      if (!ok) { J.nbr[k] = v | kPurge; continue; }
      uint64_t sc = e_nm;
      if (J.noise_cap) {
        const uint64_t key = ((uint64_t)min(n, v) << 32) | max(n, v);
        sc += __umul64hi(splitmix64(key ^ J.seed_mix), J.noise_cap + 1);   // uniform in [0, cap]
      }
      top_insert<PIMAX>(top, J.pi, sc, v);
    }
    // ---- phase 4: warp-level merges (pi rounds of shuffle argmax over list heads), then warp 0
    // merges the NW warp lists the same way; two barriers per node
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
        J.cand[(uint64_t)n * J.pi + r] = cd;
      }
    }
    if (tid == 0) ++done;
    __syncthreads();
  }
  if (tid == 0) tier_add(J.tiers, J.tier, done);
}

// feasibility + the norm=1 overflow guard
__global__ void k_score_check(const uint32_t *node_w, const uint32_t *in_mu, uint32_t lo, uint32_t hi, uint64_t omega,
                              uint64_t delta, const uint64_t *edge_off, const uint32_t *edge_w, uint32_t E, uint32_t norm,
                              uint64_t *err, unsigned long long *wsum) {
  for (uint32_t n = lo + blockIdx.x * blockDim.x + threadIdx.x; n < hi; n += gridDim.x * blockDim.x) {
    if (node_w[n] > omega) report_min(err, kErrInfeasW, n);
    if (delta != HGP_UNBOUNDED && in_mu[n] > delta) report_min(err, kErrInfeasD, n);
  }
  if (norm) {
    uint64_t s = 0;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
      s += (edge_off[e + 1] - edge_off[e]) * (uint64_t)edge_w[e];
    s = warp_sum(s);
    if (lane_id() == 0) atomicAdd(wsum, (unsigned long long)s);
  }
}

// tiers: A = 4096-slot shared table (<= 2048 entries, 32 KB), B = 16384 slots (<= 8192, 128 KB),
// W = wide accumulators (4096 slots x 16 B = 64 KB), H = global-memory tables (any size, wide)
static constexpr uint32_t kSALog = 12;   // capacity of the first tier (score_flat.cu) is 1 << (kSALog - 1)
static constexpr uint32_t kSBLog = 14, kSBThreads = 256;
static constexpr uint32_t kSWLog = 12, kSWThreads = 256;

template <int PIMAX>
hgp_status launch_score_tiers(hgp_ctx *c, ScoreJob J, uint32_t nn, uint32_t max_deg, uint32_t *lists,
                              uint32_t *counts, const uint32_t *first_list, const uint32_t *first_count) {
  hgp_status st = HGP_OK;
  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_score<kSBThreads, kModeP32, true, PIMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (8 << kSBLog) + 16);
    cudaFuncSetAttribute(k_score<kSWThreads, kModeWide, true, PIMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         16 << kSWLog);
  }
  uint32_t *bigA = lists, *wide = lists + nn, *huge = lists + 2 * (size_t)nn;
  // F (score_flat.cu): every node with |N(n)| <= 2048, packed or split accumulators; larger
  // neighbourhoods -> bigA, nodes needing 64-bit eta -> wide
  J.list = first_list; J.list_count = first_count;
  J.big_list = bigA; J.big_count = counts + 0; J.wide_list = wide; J.wide_count = counts + 1;
  const uint64_t *cv = nullptr;
  const uint2 *wmu = nullptr;
  HGP_TRY(launch_score_flat<PIMAX>(c, J, nn, J.E, &cv, &wmu));
  const uint32_t *bigL = bigA, *bigC = counts + 0;
  if (max_deg > (1u << (kSALog - 1)) && !c->opt.no_hub) {
    // big neighbourhoods: the key-partitioned tier (score_hub.cu); what it leaves -> B as before
    uint32_t hb = 0;
    HGP_TRY(read_back(c, counts + 0, 4, &hb));
    if (hb) {
      HGP_TRY(score_hub_t<PIMAX>(c, J, cv, wmu, bigA, counts + 0, hb, lists + 3 * (size_t)nn, counts + 3));
      bigL = lists + 3 * (size_t)nn; bigC = counts + 3;
    }
  }
  if (max_deg > (1u << (kSALog - 1))) {   // B: big neighbourhoods, packed (overflow -> wide)
    J.list = bigL; J.list_count = bigC; J.cap = 1u << (kSBLog - 1); J.log2s = kSBLog; J.tier = HGP_TIER_SCORE_B;
    J.big_list = huge; J.big_count = counts + 2;
    HGP_TRY(launch(c, "score_B", k_score<kSBThreads, kModeP32, true, PIMAX>, dim3(c->sm_count), dim3(kSBThreads),
                   (8u << kSBLog) + 16, J));
  }
  // W: the rest (neighbourhoods up to 2048)
  J.list = wide; J.list_count = counts + 1; J.cap = 1u << (kSWLog - 1); J.log2s = kSWLog; J.tier = HGP_TIER_SCORE_W;
  J.big_list = huge; J.big_count = counts + 2;
  HGP_TRY(launch(c, "score_W", k_score<kSWThreads, kModeWide, true, PIMAX>, dim3(c->sm_count), dim3(kSWThreads),
                 16u << kSWLog, J));
  if (max_deg > (1u << (kSWLog - 1))) {   // H: global-memory wide tables
    uint32_t lg = kSWLog;
    while ((1u << (lg - 1)) < max_deg) ++lg;
    const uint32_t ctas = c->sm_count;
    uint32_t *gtab = scratch_raw<uint32_t>(c, ((size_t)ctas * 16 << lg) / 4, &st);
    if (st) return st;
    J.list = huge; J.list_count = counts + 2; J.cap = 0xFFFFFFFFu; J.log2s = lg; J.gtab = gtab; J.tier = HGP_TIER_SCORE_H;
    HGP_TRY(launch(c, "score_H", k_score<256, kModeWide, false, PIMAX>, dim3(ctas), dim3(256), 0, J));
  }
  return HGP_OK;
}

}  // namespace hgp

using namespace hgp;

namespace hgp {

// Argument checks, feasibility and the overflow guard shared by a3 and the fused path.
// Launches k_score_check (errors are read by score_finish).
hgp_status score_prologue(hgp_ctx *c, const hgp_csr *g, uint32_t lo, uint32_t hi, const hgp_params *p, ScoreJob *J) {
  if (p->pi < 1 || p->pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "pi must be in [1,16]");
  if (p->norm > 1) return set_error(HGP_E_ARG, "norm must be 0 or 1");
  if (p->noise_cap >= (1ull << 56)) return set_error(HGP_E_ARG, "noise_cap >= 2^56");
  if (hi > g->N || lo > hi) return set_error(HGP_E_ARG, "bad neighbour range");
  hgp_status st = HGP_OK;
  const uint32_t nn = hi - lo;
  HGP_TRY(clear_errors(c));
  unsigned long long *wsum = scratch_zero<unsigned long long>(c, 1, &st);
  if (st) return st;
  const uint32_t gchk = div_up(nn > g->E ? nn : g->E, 256);
  HGP_TRY(launch(c, "score_check", k_score_check, dim3(gchk ? (gchk < 1024 ? gchk : 1024) : 1), dim3(256), 0,
                 (const uint32_t *)g->node_w, (const uint32_t *)g->in_mu, lo, hi, p->omega, p->delta,
                 (const uint64_t *)g->edge_off, (const uint32_t *)g->edge_w, g->E, p->norm, c->d_err, wsum));
  // overflow guard (reading #2): matching totals < 2^62
  unsigned __int128 tot;
  if (p->norm) {
    uint64_t ws = 0;
    HGP_TRY(read_u64(c, (const uint64_t *)wsum, &ws));
    tot = (unsigned __int128)ws << HGP_FP_SHIFT;
  } else {
    tot = (unsigned __int128)0xFFFFFFFFull << HGP_FP_SHIFT;   // sum omega < 2^32 (a1 guard)
  }
  tot += (unsigned __int128)(g->N / 2 + 1) * p->noise_cap;
  if (tot >= ((unsigned __int128)1 << 62)) return set_error(HGP_E_OVERFLOW, "score totals may exceed 2^62");
  *J = ScoreJob{};
  J->edge_off = g->edge_off; J->edge_nsrc = g->edge_nsrc; J->pins = g->pins; J->edge_w = g->edge_w;
  J->edge_mu = g->edge_mu; J->node_w = g->node_w; J->inc_off = g->inc_off; J->inc_nin = g->inc_nin;
  J->inc = g->inc; J->in_mu = g->in_mu;
  J->lo = lo; J->hi = hi;
  J->omega = p->omega; J->delta = p->delta; J->noise_cap = p->noise_cap;
  J->seed_mix = splitmix64_host(p->noise_seed);
  J->pi = p->pi; J->norm = p->norm;
  J->E = g->E;
  J->N = g->N;
  J->tiers = c->d_tiers;
  return HGP_OK;
}

hgp_status score_finish(hgp_ctx *c) {
  uint64_t err[kErrSlots];
  HGP_TRY(fetch_errors(c, err));
  if (err[kErrInfeasW] != UINT64_MAX || err[kErrInfeasD] != UINT64_MAX) {
    // the lowest node violating either constraint (size is checked before Delta)
    const uint64_t a = err[kErrInfeasW], b = err[kErrInfeasD];
    if (a <= b) return set_error(HGP_E_INFEASIBLE, "node %llu: size exceeds omega", (unsigned long long)a);
    return set_error(HGP_E_INFEASIBLE, "node %llu: inbound edges exceed delta", (unsigned long long)b);
  }
  return HGP_OK;
}

hgp_status score_run(hgp_ctx *c, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p, hgp_cand *cand,
                     const uint32_t *list, const uint32_t *list_count) {
  ScoreJob J;
  HGP_TRY(score_prologue(c, g, nb->lo, nb->hi, p, &J));
  hgp_status st = HGP_OK;
  const uint32_t nn = nb->hi - nb->lo;
  uint32_t *counts = scratch_zero<uint32_t>(c, 4, &st);
  uint32_t *lists = scratch_raw<uint32_t>(c, 4 * (size_t)(nn ? nn : 1), &st);
  if (st) return st;
  J.nb_off = nb->off; J.nbr = nb->nbr; J.cand = cand;
  if (nn) {
    if (p->pi <= 4) HGP_TRY(launch_score_tiers<4>(c, J, nn, nb->max_deg, lists, counts, list, list_count));
    else HGP_TRY(launch_score_tiers<16>(c, J, nn, nb->max_deg, lists, counts, list, list_count));
  }
  return score_finish(c);
}

hgp_status score_list_segments(hgp_ctx *c, ScoreJob J, uint32_t nn, uint32_t max_deg, const uint32_t *list,
                               const uint32_t *list_count) {
  hgp_status st = HGP_OK;
  uint32_t *counts = scratch_zero<uint32_t>(c, 4, &st);
  uint32_t *lists = scratch_raw<uint32_t>(c, 4 * (size_t)(nn ? nn : 1), &st);
  if (st) return st;
  if (J.pi <= 4) return launch_score_tiers<4>(c, J, nn, max_deg, lists, counts, list, list_count);
  return launch_score_tiers<16>(c, J, nn, max_deg, lists, counts, list, list_count);
}

}  // namespace hgp

extern "C" hgp_status hgp_score_pairs(hgp_ctx *c, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p, hgp_cand *cand) {
  if (!c || !g || !nb || !p || !cand) return set_error(HGP_E_ARG, "hgp_score_pairs: null argument");
  ApiScope scope(c);
  return score_run(c, g, nb, p, cand, nullptr, nullptr);
}
