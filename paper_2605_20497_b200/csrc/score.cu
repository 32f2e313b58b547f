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

namespace hgp {

struct ScoreJob {
  // level
  const uint64_t *edge_off;
  const uint32_t *edge_nsrc, *pins, *edge_w, *edge_mu, *node_w;
  const uint64_t *inc_off;
  const uint32_t *inc_nin, *inc, *in_mu;
  // neighbours
  uint32_t lo, hi;
  const uint64_t *nb_off;
  uint32_t *nbr;
  // params
  uint64_t omega, delta, noise_cap, seed_mix;
  uint32_t pi, norm;
  hgp_cand *cand;
  // scheduling
  const uint32_t *list;        // nodes (nullptr: all of [lo,hi) with degree <= max_deg_here)
  const uint32_t *list_count;
  uint32_t max_deg_here;       // tier capacity in neighbour entries
  uint32_t log2s;
  uint32_t *gtab;              // global tables when !SMEM: per CTA (4 + 8 + 4) << log2s bytes
};

struct Top {   // best-first list of (score, id); empty entries have id == kNone
  uint64_t s[HGP_MAX_PI];
  uint32_t id[HGP_MAX_PI];
};

__device__ __forceinline__ bool better(uint64_t s1, uint32_t i1, uint64_t s2, uint32_t i2) {
  // (score desc, id desc); an empty entry (kNone) is worse than any real one
  if (i2 == kNone) return i1 != kNone;
  if (i1 == kNone) return false;
  return s1 > s2 || (s1 == s2 && i1 > i2);
}

__device__ __forceinline__ void top_insert(Top &t, uint32_t pi, uint64_t s, uint32_t id) {
#pragma unroll
  for (int i = 0; i < HGP_MAX_PI; ++i) {
    if (i < (int)pi && better(s, id, t.s[i], t.id[i])) {
      uint64_t ts = t.s[i]; uint32_t ti = t.id[i];
      t.s[i] = s; t.id[i] = id;
      s = ts; id = ti;
    }
  }
}

template <int THREADS, bool SMEM>
__global__ void __launch_bounds__(THREADS) k_score(ScoreJob J) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint64_t red_s[THREADS / 32];
  __shared__ uint32_t red_i[THREADS / 32], red_t[THREADS / 32];
  __shared__ uint32_t s_win;
  constexpr uint32_t NW = THREADS / 32;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t log2s = J.log2s, S = 1u << log2s;
  unsigned char *base = SMEM ? dyn : reinterpret_cast<unsigned char *>(J.gtab) + ((size_t)blockIdx.x * 16 << log2s);
  uint64_t *eta = reinterpret_cast<uint64_t *>(base);
  uint32_t *keys = reinterpret_cast<uint32_t *>(base + ((size_t)8 << log2s));
  uint32_t *inter = reinterpret_cast<uint32_t *>(base + ((size_t)12 << log2s));
  const uint32_t total = J.list_count ? *J.list_count : J.hi - J.lo;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t n = J.list ? J.list[t] : J.lo + t;
    const uint64_t b0 = J.nb_off[n - J.lo], b1 = J.nb_off[n - J.lo + 1];
    if (!J.list && b1 - b0 > J.max_deg_here) continue;           // handled by a larger tier (uniform)
    for (uint32_t i = tid; i < S; i += THREADS) { keys[i] = kEmpty; eta[i] = 0; inter[i] = 0; }
    __syncthreads();
    for (uint64_t k = b0 + tid; k < b1; k += THREADS) {          // bins = unflagged neighbours
      const uint32_t v = J.nbr[k];
      if (!(v & kPurge)) hs_insert(keys, log2s, v);
    }
    __syncthreads();
    // traverse I(n): warp per incident edge, lanes over its pins (Eq.4 nesting)
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    for (uint64_t k = i0 + w; k < i1; k += NW) {
      const uint32_t e = J.inc[k];
      const uint64_t a = J.edge_off[e], b = J.edge_off[e + 1], s = a + J.edge_nsrc[e];
      const uint64_t we = (uint64_t)J.edge_w[e] << HGP_FP_SHIFT;
      const uint64_t ce = J.norm ? we : we / (b - a);
      const uint32_t mu_in = k < iin ? J.edge_mu[e] : 0u;       // e in in(n)
      for (uint64_t j = a + lane; j < b; j += 32) {
        const uint32_t m = J.pins[j];
        if (m == n) continue;
        const uint32_t slot = hs_find(keys, log2s, m);
        if (slot == kNone) continue;                              // purged neighbour
        atomicAdd(reinterpret_cast<unsigned long long *>(&eta[slot]), (unsigned long long)ce);
        if (mu_in && j >= s) atomicAdd(&inter[slot], mu_in);
      }
    }
    __syncthreads();
    // validity, purge flags, noise, per-thread top-pi
    Top top;
#pragma unroll
    for (int i = 0; i < HGP_MAX_PI; ++i) { top.s[i] = 0; top.id[i] = kNone; }
    const uint64_t wn = J.node_w[n], inn = J.in_mu[n];
    for (uint64_t k = b0 + tid; k < b1; k += THREADS) {
      const uint32_t v = J.nbr[k];
      if (v & kPurge) continue;
      const uint32_t slot = hs_find(keys, log2s, v);
      const uint64_t uni = inn + J.in_mu[v] - inter[slot];        // |in(n) ∪ in(m)|
      const bool ok = wn + J.node_w[v] <= J.omega && (J.delta == HGP_UNBOUNDED || uni <= J.delta);
      if (!ok) { J.nbr[k] = v | kPurge; continue; }
      uint64_t sc = eta[slot];
      if (J.noise_cap) {
        const uint64_t key = ((uint64_t)min(n, v) << 32) | max(n, v);
        sc += splitmix64(key ^ J.seed_mix) % (J.noise_cap + 1);
      }
      top_insert(top, J.pi, sc, v);
    }
    // CTA-wide merge of the per-thread lists: pi rounds of argmax over list heads
    uint32_t head = 0;
    for (uint32_t r = 0; r < J.pi; ++r) {
      uint64_t hs = 0;
      uint32_t hid = kNone;
#pragma unroll
      for (int i = 0; i < HGP_MAX_PI; ++i)
        if (i == (int)head) { hs = top.s[i]; hid = top.id[i]; }
      uint32_t who = tid;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t os = __shfl_xor_sync(0xFFFFFFFFu, hs, o);
        const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, hid, o);
        const uint32_t ow = __shfl_xor_sync(0xFFFFFFFFu, who, o);
        if (better(os, oi, hs, hid)) { hs = os; hid = oi; who = ow; }
      }
      if (lane == 0) { red_s[w] = hs; red_i[w] = hid; red_t[w] = who; }
      __syncthreads();
      if (tid == 0) {
        uint64_t bs = red_s[0];
        uint32_t bi = red_i[0], bt = red_t[0];
        for (uint32_t q = 1; q < NW; ++q)
          if (better(red_s[q], red_i[q], bs, bi)) { bs = red_s[q]; bi = red_i[q]; bt = red_t[q]; }
        hgp_cand cd;
        cd.id = bi; cd.pad = 0; cd.score = bi == kNone ? 0 : bs;
        J.cand[(uint64_t)n * J.pi + r] = cd;
        s_win = bi == kNone ? kNone : bt;
      }
      __syncthreads();
      if (s_win == tid) ++head;
    }
    __syncthreads();
  }
}

__global__ void k_score_classify(const uint64_t *nb_off, uint32_t lo, uint32_t hi, uint32_t capA, uint32_t capB,
                                 uint32_t *listB, uint32_t *listC, uint32_t *counts) {
  for (uint32_t n = lo + blockIdx.x * blockDim.x + threadIdx.x; n < hi; n += gridDim.x * blockDim.x) {
    const uint64_t d = nb_off[n - lo + 1] - nb_off[n - lo];
    if (d > capA) {
      if (d <= capB) listB[atomicAdd(&counts[0], 1u)] = n;
      else listC[atomicAdd(&counts[1], 1u)] = n;
    }
  }
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

static constexpr uint32_t kSALog = 11, kSAThreads = 128;   // 2048 slots x 16 B = 32 KB, <= 1024 entries
static constexpr uint32_t kSBLog = 13, kSBThreads = 256;   // 8192 slots = 128 KB, <= 4096 entries

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_score_pairs(hgp_ctx *c, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p, hgp_cand *cand) {
  if (!c || !g || !nb || !p || !cand) return set_error(HGP_E_ARG, "hgp_score_pairs: null argument");
  if (p->pi < 1 || p->pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "pi must be in [1,16]");
  if (p->norm > 1) return set_error(HGP_E_ARG, "norm must be 0 or 1");
  if (p->noise_cap >= (1ull << 56)) return set_error(HGP_E_ARG, "noise_cap >= 2^56");
  if (nb->hi > g->N || nb->lo > nb->hi) return set_error(HGP_E_ARG, "bad neighbour range");
  ApiScope scope(c);
  hgp_status st = HGP_OK;
  const uint32_t lo = nb->lo, hi = nb->hi, nn = hi - lo;
  HGP_TRY(clear_errors(c));
  uint32_t *counts = scratch_zero<uint32_t>(c, 4, &st);
  unsigned long long *wsum = scratch_zero<unsigned long long>(c, 1, &st);
  if (st) return st;
  const uint32_t gchk = div_up(nn > g->E ? nn : g->E, 256);
  HGP_TRY(launch(c, "score_check", k_score_check, dim3(gchk ? (gchk < 1024 ? gchk : 1024) : 1), dim3(256), 0,
                 (const uint32_t *)g->node_w, (const uint32_t *)g->in_mu, lo, hi, p->omega, p->delta,
                 (const uint64_t *)g->edge_off, (const uint32_t *)g->edge_w, g->E, p->norm, c->d_err, wsum));
  // overflow guard (reading #2): matching totals < 2^62
  {
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
  }
  ScoreJob J{};
  J.edge_off = g->edge_off; J.edge_nsrc = g->edge_nsrc; J.pins = g->pins; J.edge_w = g->edge_w;
  J.edge_mu = g->edge_mu; J.node_w = g->node_w; J.inc_off = g->inc_off; J.inc_nin = g->inc_nin;
  J.inc = g->inc; J.in_mu = g->in_mu;
  J.lo = lo; J.hi = hi; J.nb_off = nb->off; J.nbr = nb->nbr;
  J.omega = p->omega; J.delta = p->delta; J.noise_cap = p->noise_cap;
  J.seed_mix = splitmix64_host(p->noise_seed);
  J.pi = p->pi; J.norm = p->norm; J.cand = cand;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_score<kSAThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 << kSALog);
    cudaFuncSetAttribute(k_score<kSBThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 << kSBLog);
    attr = true;
  }
  const uint32_t capA = 1u << (kSALog - 1), capB = 1u << (kSBLog - 1);
  // tier A: every node whose neighbourhood fits 1024 entries
  J.list = nullptr; J.list_count = nullptr; J.max_deg_here = capA; J.log2s = kSALog;
  const uint32_t gA = nn < 64u * c->sm_count ? nn : 64u * c->sm_count;
  HGP_TRY(launch(c, "score_A", k_score<kSAThreads, true>, dim3(gA), dim3(kSAThreads), 16u << kSALog, J));
  if (nb->max_deg > capA) {
    uint32_t *lists = scratch_raw<uint32_t>(c, 2 * (size_t)nn, &st);
    if (st) return st;
    HGP_TRY(launch(c, "score_classify", k_score_classify, dim3(div_up(nn, 256) < 1024 ? div_up(nn, 256) : 1024),
                   dim3(256), 0, (const uint64_t *)nb->off, lo, hi, capA, capB, lists, lists + nn, counts));
    J.list = lists; J.list_count = counts; J.max_deg_here = capB; J.log2s = kSBLog;
    HGP_TRY(launch(c, "score_B", k_score<kSBThreads, true>, dim3(c->sm_count), dim3(kSBThreads), 16u << kSBLog, J));
    if (nb->max_deg > capB) {
      uint32_t lg = kSBLog;
      while ((1u << (lg - 1)) < nb->max_deg) ++lg;
      const uint32_t ctas = c->sm_count;
      uint32_t *gtab = scratch_raw<uint32_t>(c, ((size_t)ctas * 16 << lg) / 4, &st);
      if (st) return st;
      J.list = lists + nn; J.list_count = counts + 1; J.max_deg_here = 1u << (lg - 1); J.log2s = lg; J.gtab = gtab;
      HGP_TRY(launch(c, "score_C", k_score<256, false>, dim3(ctas), dim3(256), 0, J));
    }
  }
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
