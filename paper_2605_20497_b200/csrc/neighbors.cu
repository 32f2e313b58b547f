// neighbors.cu — a2: materialise N(n) = (U_{e in I(n)} e) \ {n}.
//
// One CTA per node deduplicates the pins of its incident hyperedges in an open-addressing
// hash set (shared memory; global memory for giant neighbourhoods), then appends the unique
// ids to a pool at an atomically reserved offset; a scan of the counts and a pack give the
// CSR. Segments are sets (hash order), see include/hgp.h.
#include "csr_impl.cuh"
#include "pack.cuh"
#include "hashset.cuh"
#include "scan.cuh"

namespace hgp {

struct NbrJob {
  const uint64_t *inc_off;
  const uint32_t *inc;
  const uint64_t *edge_off;
  const uint32_t *pins;
  uint32_t lo;
  const uint32_t *list;        // nodes to process (nullptr: lo + t for t < nall)
  const uint32_t *list_count;  // device count of list (nullptr: nall)
  uint32_t nall;
  uint32_t log2s;              // table size
  uint32_t cap;                // max uniques before declaring overflow
  uint32_t *gtab;              // global tables (one per CTA) when not in smem
  uint32_t *pool;
  uint64_t pool_cap;
  unsigned long long *pool_cursor;
  uint64_t *start;             // [hi-lo]
  uint32_t *cnt;               // [hi-lo]
  uint32_t *ovf_list, *ovf_count;    // table overflow -> next tier
  uint32_t *pool_list, *pool_count;  // pool overflow -> rerun after growing the pool
  uint64_t start_bias;               // added to every start written (pool base differs from the view's)
  unsigned long long *tiers;         // work counters (hgp_tier_counts)
  int tier;
};

template <int THREADS, bool SMEM>
__global__ void __launch_bounds__(THREADS) k_nbrs(NbrJob J) {
  extern __shared__ uint32_t dyn[];
  __shared__ uint32_t s_cnt;
  __shared__ uint32_t s_state;    // 0 ok, 1 table overflow, 2 pool overflow
  __shared__ unsigned long long s_start;
  constexpr uint32_t NW = THREADS / 32;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t *tab = SMEM ? dyn : J.gtab + ((size_t)blockIdx.x << J.log2s);
  const uint32_t total = J.list_count ? *J.list_count : J.nall;
  uint32_t done = 0;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t n = J.list ? J.list[t] : J.lo + t;
    // global tables: only nextpow2(2 (bound + 1) + margin) slots of the CTA's region, bound =
    // sum over I(n) of (|e| - 1), so clearing and sweeping cost what the node needs
    uint32_t nlog = J.log2s;
    if (!SMEM) {
      uint64_t bsum = 0;
      for (uint64_t k = J.inc_off[n] + tid; k < J.inc_off[n + 1]; k += THREADS) {
        const uint32_t e = J.inc[k];
        bsum += J.edge_off[e + 1] - J.edge_off[e] - 1;
      }
      bsum = warp_sum(bsum);
      if (tid == 0) s_start = 0;
      __syncthreads();
      if (lane == 0 && bsum) atomicAdd(&s_start, (unsigned long long)bsum);
      __syncthreads();
      const uint64_t need = 2 * (s_start + 1) + 128 * NW;
      __syncthreads();                                             // s_start is reused below
      nlog = 6;
      while ((1ull << nlog) < need && nlog < J.log2s) ++nlog;
    }
    const uint32_t Sn = 1u << nlog;
    for (uint32_t i = tid; i < Sn / 4; i += THREADS)
      reinterpret_cast<uint4 *>(tab)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    if (tid == 0) { s_cnt = 0; s_state = 0; }
    __syncthreads();
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1];
    volatile uint32_t *vcnt = &s_cnt;
    const uint32_t tab_s = SMEM ? opaque_u32(smem_u32addr(tab)) : 0u;
    const uint32_t hmask = Sn - 1;
    bool stop = false;
    uint32_t nins = 0;                                             // new keys, flushed per block
    // a warp loads the offsets of 32 incident edges at once (lane = edge), then walks them with
    // 128 pins in flight per iteration (4 per lane)
    for (uint64_t kb = i0 + w; kb < i1 && !stop; kb += (uint64_t)NW * 32) {   // round-robin over warps
      const uint64_t k = kb + (uint64_t)NW * lane;
      uint64_t a = 0;
      uint32_t len = 0;
      if (k < i1) {
        const uint32_t e = J.inc[k];
        a = J.edge_off[e];
        len = (uint32_t)(J.edge_off[e + 1] - a);
      }
      const uint32_t cnt = (uint32_t)min((uint64_t)32, (i1 - kb + NW - 1) / NW);
      for (uint32_t j = 0; j < cnt && !stop; ++j) {
        const uint64_t aj = __shfl_sync(0xFFFFFFFFu, a, j);
        const uint32_t lj = __shfl_sync(0xFFFFFFFFu, len, j);
        const uint32_t *pj = J.pins + aj;
        for (uint32_t b4 = 0; b4 < lj; b4 += 128) {
          // warp-uniform decision: lanes may reach this point at different times (independent
          // thread scheduling), so vote instead of trusting each lane's own read
          if (__any_sync(0xFFFFFFFFu, *vcnt >= J.cap)) { stop = true; break; }
          uint32_t m[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t idx = b4 + u * 32 + lane;
            m[u] = idx < lj ? __ldg(pj + idx) : n;
          }
          // first probes of the 4 pins issued back to back (ILP); a hit (the common case: most
          // pins repeat a neighbour already seen) needs nothing else
          if constexpr (!SMEM) {   // global-memory table: generic atomics
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (m[u] != n && hs_insert(tab, nlog, m[u])) ++nins;
          } else {
          uint32_t sl[4], kk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) sl[u] = hash_slot(m[u], nlog);
#pragma unroll
          for (int u = 0; u < 4; ++u) kk[u] = lds_hint_u32(tab_s + 4 * sl[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (m[u] == n || kk[u] == m[u]) continue;
            uint32_t slot = sl[u], k2 = kk[u];
            while (true) {
              if (k2 == kEmpty) {
                k2 = cas_u32(tab_s + 4 * slot, kEmpty, m[u]);
                if (k2 == kEmpty) { ++nins; break; }
              }
              if (k2 == m[u]) break;
              slot = (slot + 1) & hmask;
              k2 = lds_hint_u32(tab_s + 4 * slot);
            }
          }
          }
          const uint32_t tins = __reduce_add_sync(0xFFFFFFFFu, nins);
          if (lane == 0 && tins) atomicAdd(&s_cnt, tins);
          nins = 0;
        }
      }
    }
    if (stop && lane == 0) s_state = 1;
    __syncthreads();
    const uint32_t count = s_cnt;
    if (s_state == 0 && tid == 0) {
      unsigned long long st = atomicAdd(J.pool_cursor, (unsigned long long)count);
      s_start = st;
      if (st + count > J.pool_cap) s_state = 2;
    }
    __syncthreads();
    if (s_state == 1) {
      if (tid == 0) J.ovf_list[atomicAdd(J.ovf_count, 1u)] = n;
    } else if (s_state == 2) {
      if (tid == 0) J.pool_list[atomicAdd(J.pool_count, 1u)] = n;
    } else {
      // compact the occupied slots: warps sweep 32 consecutive slots at a time (conflict-free)
      if (tid == 0) s_cnt = 0;
      __syncthreads();
      const uint32_t lt = (1u << lane) - 1;
      for (uint32_t sb = w * 32; sb < Sn; sb += NW * 32) {
        const uint32_t v = tab[sb + lane];
        const bool has = v != kEmpty;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, has);
        if (!bal) continue;
        uint32_t wpos = 0;
        if (lane == 0) wpos = atomicAdd(&s_cnt, __popc(bal));
        wpos = __shfl_sync(0xFFFFFFFFu, wpos, 0);
        if (has) J.pool[s_start + wpos + __popc(bal & lt)] = v;
      }
      if (tid == 0) { J.start[n - J.lo] = s_start + J.start_bias; J.cnt[n - J.lo] = count; ++done; }
    }
    __syncthreads();
  }
  if (tid == 0) tier_add(J.tiers, J.tier, done);
}

// bound_n = min(N-1, sum_{e in I(n)} (|e|-1)) for the listed nodes -> atomicMax
__global__ void k_nbr_bound(const uint64_t *inc_off, const uint32_t *inc, const uint64_t *edge_off,
                            const uint32_t *list, const uint32_t *count, uint32_t N, unsigned long long *mx) {
  const uint32_t total = *count;
  for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < total; t += gridDim.x * (blockDim.x >> 5)) {
    const uint32_t n = list[t];
    uint64_t s = 0;
    for (uint64_t k = inc_off[n] + lane_id(); k < inc_off[n + 1]; k += 32) {
      const uint32_t e = inc[k];
      s += edge_off[e + 1] - edge_off[e] - 1;
    }
    s = warp_sum(s);
    if (s > N - 1) s = N - 1;
    if (lane_id() == 0) atomicMax(mx, (unsigned long long)s);
  }
}

__global__ void k_seg_pack_flat(const uint32_t *pool, const uint64_t *start, const uint32_t *cnt, const uint64_t *off,
                                uint32_t nn, uint64_t V, uint32_t *nbr, unsigned int *maxdeg) {
  const uint32_t lane = lane_id();
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t mx = 0;                                                  // max segment: grid-stride over t
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += gridDim.x * blockDim.x) mx = max(mx, cnt[t]);
  mx = warp_max(mx);
  if (lane == 0 && mx) atomicMax(maxdeg, mx);
  const uint64_t lo = V * wid / W, hi = V * (wid + 1) / W;
  if (lo >= hi) return;
  uint32_t a = 0, b = nn;                                           // last t with off[t] <= lo
  while (b - a > 1) {
    const uint32_t m = (a + b) >> 1;
    if (off[m] <= lo) a = m; else b = m;
  }
  uint64_t pos = lo;
  for (uint32_t t = a; pos < hi; ++t) {
    const uint64_t s0 = off[t], s1 = off[t + 1];
    if (s1 <= pos) continue;
    const uint32_t i0 = (uint32_t)(pos - s0), i1 = (uint32_t)((s1 < hi ? s1 : hi) - s0);
    const uint32_t *src = pool + start[t];
    uint32_t *dst = nbr + s0;
    for (uint32_t j0 = i0; j0 < i1; j0 += 128) {                    // 4 loads in flight per lane
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { const uint32_t i = j0 + u * 32 + lane; v[u] = i < i1 ? src[i] : 0u; }
#pragma unroll
      for (int u = 0; u < 4; ++u) { const uint32_t i = j0 + u * 32 + lane; if (i < i1) dst[i] = v[u]; }
    }
    pos = s0 + i1;
  }
}

__global__ void k_edge_pairs(const uint64_t *edge_off, uint32_t E, unsigned long long *T) {
  uint64_t s = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint64_t d = edge_off[e + 1] - edge_off[e];
    s += d * (d - 1);
  }
  s = warp_sum(s);
  if (lane_id() == 0) atomicAdd(T, (unsigned long long)s);
}

void free_nbrs(hgp_ctx *c, hgp_nbrs *nb) {
  if (!nb) return;
  c->dfree(nb->off, 8 * ((size_t)(nb->hi - nb->lo) + 1));
  c->dfree(nb->nbr, 4 * nb->V);
  memset(nb, 0, sizeof(*nb));
}

static constexpr uint32_t kT1Log = 12, kT1Threads = 128;   // 16 KB table + 8 KB list, <= 1536 uniques
static constexpr uint32_t kT2Log = 15, kT2Threads = 256;   // 128 KB table + 64 KB list

__global__ void k_list_bound_sum(const uint64_t *inc_off, const uint32_t *inc, const uint64_t *edge_off,
                                 const uint32_t *list, const uint32_t *count, uint32_t N, unsigned long long *sum,
                                 unsigned long long *mx) {
  const uint32_t total = *count;
  uint64_t acc = 0, m = 0;
  for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < total; t += gridDim.x * (blockDim.x >> 5)) {
    const uint32_t n = list[t];
    uint64_t s = 0;
    for (uint64_t k = inc_off[n] + lane_id(); k < inc_off[n + 1]; k += 32) {
      const uint32_t e = inc[k];
      s += edge_off[e + 1] - edge_off[e] - 1;
    }
    s = warp_sum(s);
    if (s > N - 1) s = N - 1;
    acc += s;
    m = s > m ? s : m;
  }
  if (lane_id() == 0) { atomicAdd(sum, (unsigned long long)acc); atomicMax(mx, (unsigned long long)m); }
}

static constexpr uint32_t kT1LogL = 12, kT1ThreadsL = 128;
static constexpr uint32_t kT2LogL = 15, kT2ThreadsL = 256;

// a2 for the nodes of a device list (hcount = its host-known length): N(n) into a fresh pool
// sized min(exact bound, 8 P + hcount), with bound = sum_n min(sum_{e in I(n)} (|e|-1), N-1); a
// too-short pool is regrown once to the exact total (the cursor). start/cnt are indexed n - lo,
// start relative to `base`; *max_deg_out = an upper bound of the counts.
hgp_status nbrs_for_list(hgp_ctx *c, const hgp_csr *g, uint32_t lo, const uint32_t *list, const uint32_t *list_count,
                         uint32_t hcount, const uint32_t *base, uint64_t *start, uint32_t *cnt, uint32_t *max_deg_out) {
  hgp_status st = HGP_OK;
  unsigned long long *misc = scratch_zero<unsigned long long>(c, 4, &st);   // sum, max, cursor, -
  uint32_t *counters = scratch_zero<uint32_t>(c, 8, &st);
  uint32_t *list1 = scratch_raw<uint32_t>(c, hcount ? hcount : 1, &st);
  uint32_t *list2 = scratch_raw<uint32_t>(c, hcount ? hcount : 1, &st);
  uint32_t *plist = scratch_raw<uint32_t>(c, hcount ? hcount : 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "nbr_list_bound", k_list_bound_sum, dim3(c->sm_count), dim3(256), 0, (const uint64_t *)g->inc_off,
                 (const uint32_t *)g->inc, (const uint64_t *)g->edge_off, list, list_count, g->N, misc, misc + 1));
  uint64_t hb[2];
  HGP_TRY(read_back(c, misc, 16, hb));
  *max_deg_out = (uint32_t)hb[1];
  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_nbrs<kT1ThreadsL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << kT1LogL);
    cudaFuncSetAttribute(k_nbrs<kT2ThreadsL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << kT2LogL);
  }
  uint32_t *gtab = nullptr;
  uint32_t lg = 1;
  const bool t3 = hb[1] + 1 > (1u << (kT2LogL - 1)) - 128 * (kT2ThreadsL / 32);
  if (t3) {   // tier 3: global tables
    while ((1ull << lg) < 2 * (hb[1] + 1) + 128 * 8) ++lg;
    gtab = scratch_raw<uint32_t>(c, (size_t)c->sm_count << lg, &st);
    if (st) return st;
  }
  uint64_t pool_cap = hb[0] + hcount < (1ull << 34) ? hb[0] + hcount : (1ull << 34);   // the exact bound
  for (int attempt = 0;; ++attempt) {
    if (pool_cap == 0) pool_cap = 1;
    uint32_t *pool = scratch_raw<uint32_t>(c, pool_cap, &st);
    if (st) return st;
    HGP_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(uint32_t), c->stream));
    HGP_CUDA(cudaMemsetAsync(misc + 2, 0, sizeof(unsigned long long), c->stream));
    NbrJob J{};
    J.inc_off = g->inc_off; J.inc = g->inc; J.edge_off = g->edge_off; J.pins = g->pins;
    J.lo = lo; J.pool = pool; J.pool_cap = pool_cap; J.pool_cursor = misc + 2;
    J.start_bias = (uint64_t)(pool - base);
    J.start = start; J.cnt = cnt; J.pool_list = plist; J.pool_count = counters + 5;
    J.list = list; J.list_count = list_count;
    J.tiers = c->d_tiers; J.tier = HGP_TIER_NBRS_1; J.log2s = kT1LogL; J.cap = (1u << (kT1LogL - 1)) - 128 * (kT1ThreadsL / 32);
    J.ovf_list = list1; J.ovf_count = counters + 0;
    HGP_TRY(launch(c, "nbrs_list_t1", k_nbrs<kT1ThreadsL, true>, dim3(8u * c->sm_count), dim3(kT1ThreadsL),
                   4u << kT1LogL, J));
    J.list = list1; J.list_count = counters + 0;
    J.tiers = c->d_tiers; J.tier = HGP_TIER_NBRS_2; J.log2s = kT2LogL; J.cap = (1u << (kT2LogL - 1)) - 128 * (kT2ThreadsL / 32);
    J.ovf_list = list2; J.ovf_count = counters + 1;
    HGP_TRY(launch(c, "nbrs_list_t2", k_nbrs<kT2ThreadsL, true>, dim3(c->sm_count), dim3(kT2ThreadsL), 4u << kT2LogL, J));
    if (t3) {
      J.list = list2; J.list_count = counters + 1; J.log2s = lg; J.cap = 0xFFFFFFFFu; J.gtab = gtab; J.tier = HGP_TIER_NBRS_3;
      J.ovf_list = list1; J.ovf_count = counters + 4;   // cannot overflow: table >= 2 (bound + 1)
      HGP_TRY(launch(c, "nbrs_list_t3", k_nbrs<256, false>, dim3(c->sm_count), dim3(256), 0, J));
    }
    uint32_t hc[8];
    HGP_TRY(read_back(c, counters, sizeof(hc), hc));
    if (hc[5] == 0) return HGP_OK;
    if (attempt == 1) return set_error(HGP_E_INTERNAL, "nbrs_for_list: pool sizing failed");
    uint64_t cur = 0;
    HGP_TRY(read_u64(c, (const uint64_t *)(misc + 2), &cur));
    pool_cap = cur;
  }
}

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_unique_neighbors(hgp_ctx *c, const hgp_csr *g, uint32_t lo, uint32_t hi, hgp_nbrs *out) {
  if (!c || !g || !out || lo > hi || hi > g->N) return set_error(HGP_E_ARG, "hgp_unique_neighbors: bad argument");
  ApiScope scope(c);
  memset(out, 0, sizeof(*out));
  hgp_status st = HGP_OK;
  const uint32_t nn = hi - lo;
  out->lo = lo;
  out->hi = hi;
  out->off = dalloc_n<uint64_t>(c, (size_t)nn + 1, &st);
  if (st) return st;
  if (nn == 0) {
    HGP_CUDA(cudaMemsetAsync(out->off, 0, 8, c->stream));
    out->nbr = dalloc_n<uint32_t>(c, 1, &st);
    return st;
  }
  // pool capacity: T = sum_e |e|(|e|-1) >= total pre-dedup candidates
  unsigned long long *misc = scratch_zero<unsigned long long>(c, 4, &st);   // T, cursor, bound, -
  uint32_t *counters = scratch_zero<uint32_t>(c, 8, &st);                  // ovf1, ovf2, poolovf, maxdeg
  uint64_t *start = scratch_raw<uint64_t>(c, nn, &st);
  uint32_t *cnt = scratch_raw<uint32_t>(c, nn, &st);
  uint32_t *list1 = scratch_raw<uint32_t>(c, nn, &st);
  uint32_t *list2 = scratch_raw<uint32_t>(c, nn, &st);
  uint32_t *plist = scratch_raw<uint32_t>(c, nn, &st);
  if (st) return st;
  HGP_TRY(launch(c, "edge_pairs", k_edge_pairs, dim3(g->E ? (div_up(g->E, 256) < 1024 ? div_up(g->E, 256) : 1024) : 0),
                 dim3(256), 0, (const uint64_t *)g->edge_off, g->E, misc));
  uint64_t T = 0;
  HGP_TRY(read_u64(c, (const uint64_t *)misc, &T));
  // T bounds the total exactly (|N(n)| <= sum over I(n) of (|e| - 1)); a smaller estimate makes
  // power-law inputs (V ~ T) pay a second full pass. At most 2^34 entries; beyond, the retry.
  uint64_t pool_cap = T + nn < (1ull << 34) ? T + nn : (1ull << 34);
  if (pool_cap == 0) pool_cap = 1;
  uint32_t *pool = scratch_raw<uint32_t>(c, pool_cap, &st);
  if (st) return st;

  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_nbrs<kT1Threads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << kT1Log);
    cudaFuncSetAttribute(k_nbrs<kT2Threads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << kT2Log);
  }
  // Run the three tiers with a given pool; returns pool-overflow count and the pool cursor
  // (= exact total of unique entries once every node has deduplicated).
  auto run_tiers = [&](uint32_t *pool, uint64_t pool_cap, uint32_t *n_pool_ovf, uint64_t *cursor) -> hgp_status {
    HGP_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(uint32_t), c->stream));
    HGP_CUDA(cudaMemsetAsync(misc + 1, 0, 3 * sizeof(unsigned long long), c->stream));
    NbrJob J{};
    J.inc_off = g->inc_off; J.inc = g->inc; J.edge_off = g->edge_off; J.pins = g->pins;
    J.lo = lo; J.pool = pool; J.pool_cap = pool_cap; J.pool_cursor = misc + 1;
    J.start = start; J.cnt = cnt; J.pool_list = plist; J.pool_count = counters + 2;
    // tier 1: every node, 16 KB shared table
    J.list = nullptr; J.list_count = nullptr; J.nall = nn;
    J.tiers = c->d_tiers; J.tier = HGP_TIER_NBRS_1; J.log2s = kT1Log; J.cap = (1u << (kT1Log - 1)) - 128 * (kT1Threads / 32);
    J.ovf_list = list1; J.ovf_count = counters + 0;
    const uint32_t grid1 = nn < 32u * c->sm_count ? nn : 32u * c->sm_count;
    HGP_TRY(launch(c, "nbrs_t1", k_nbrs<kT1Threads, true>, dim3(grid1), dim3(kT1Threads), 4u << kT1Log, J));
    // tier 2: 128 KB shared table for the overflowed nodes (grid-stride over a device count)
    J.list = list1; J.list_count = counters + 0;
    J.tiers = c->d_tiers; J.tier = HGP_TIER_NBRS_2; J.log2s = kT2Log; J.cap = (1u << (kT2Log - 1)) - 128 * (kT2Threads / 32);
    J.ovf_list = list2; J.ovf_count = counters + 1;
    HGP_TRY(launch(c, "nbrs_t2", k_nbrs<kT2Threads, true>, dim3(c->sm_count), dim3(kT2Threads), 4u << kT2Log, J));
    uint32_t hc[4];
    HGP_TRY(read_back(c, counters, 16, hc));
    if (hc[1]) {   // tier 3: global-memory tables sized from the neighbourhood bound
      HGP_TRY(launch(c, "nbr_bound", k_nbr_bound, dim3(c->sm_count), dim3(256), 0, (const uint64_t *)g->inc_off,
                     (const uint32_t *)g->inc, (const uint64_t *)g->edge_off, (const uint32_t *)list2,
                     (const uint32_t *)(counters + 1), g->N, misc + 2));
      uint64_t mb = 0;
      HGP_TRY(read_u64(c, (const uint64_t *)(misc + 2), &mb));
      uint32_t lg = 1;
      while ((1ull << lg) < 2 * (mb + 1) + 128 * 8) ++lg;
      const uint32_t ctas = hc[1] < (uint32_t)c->sm_count ? hc[1] : (uint32_t)c->sm_count;
      uint32_t *gtab = scratch_raw<uint32_t>(c, (size_t)ctas << lg, &st);
      if (st) return st;
      J.list = list2; J.list_count = counters + 1; J.log2s = lg; J.cap = 0xFFFFFFFFu; J.gtab = gtab; J.tier = HGP_TIER_NBRS_3;
      J.ovf_list = list1; J.ovf_count = counters + 4;   // cannot overflow: table >= 2 (bound + 1)
      HGP_TRY(launch(c, "nbrs_t3", k_nbrs<256, false>, dim3(ctas), dim3(256), 0, J));
      HGP_TRY(read_back(c, counters, 16, hc));
    }
    *n_pool_ovf = hc[2];
    return read_u64(c, (const uint64_t *)(misc + 1), cursor);
  };
  uint32_t n_pool_ovf = 0;
  uint64_t cursor = 0;
  HGP_TRY(run_tiers(pool, pool_cap, &n_pool_ovf, &cursor));
  for (int attempt = 0; n_pool_ovf; ++attempt) {   // estimate too short: the cursor holds the exact total
    if (attempt == 2) return set_error(HGP_E_INTERNAL, "hgp_unique_neighbors: pool sizing failed");
    pool_cap = cursor;
    pool = scratch_raw<uint32_t>(c, pool_cap, &st);
    if (st) return st;
    HGP_TRY(run_tiers(pool, pool_cap, &n_pool_ovf, &cursor));
  }
  uint64_t V = 0;
  HGP_TRY(scan_exclusive(c, InU32{cnt}, nn, out->off, &V));
  out->V = V;
  out->nbr = dalloc_n<uint32_t>(c, V, &st);
  if (st) { free_nbrs(c, out); return st; }
  unsigned int *d_max = counters + 3;
  hgp_status s = launch(c, "nbr_pack", k_seg_pack_flat, dim3(8u * c->sm_count), dim3(256), 0, (const uint32_t *)pool,
                        (const uint64_t *)start, (const uint32_t *)cnt, (const uint64_t *)out->off, nn, V, out->nbr, d_max);
  if (s) { free_nbrs(c, out); return s; }
  uint32_t mx = 0;
  s = read_back(c, d_max, 4, &mx);
  if (s) { free_nbrs(c, out); return s; }
  out->max_deg = mx;
  return HGP_OK;
}

extern "C" void hgp_nbrs_free(hgp_ctx *c, hgp_nbrs *nb) {
  if (c && nb) { DeviceGuard dg(c->device); free_nbrs(c, nb); }
}
