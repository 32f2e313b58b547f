// hub.cu — hub nodes of the fused level-0 a2 + a3.
//
// A hub's neighbourhood overflows every shared-memory table (power-law inputs: C3 has ~3,400 nodes
// with 8,192 < b(n) <= 10^6 pin visits, b(n) = sum over I(n) of (|e| - 1) >= |N(n)|). One CTA
// probing a global-memory table for such a node is bound by atomic latency (measured: a2 tier 3
// + a3 tier H = 180 ms on C3). Here a hub's visits are split by a hash of the neighbour id into
// k(n) = ceil(b(n) / kHubPart) partitions, so that every partition fits the A-size shared table:
//   plan     per hub: b(n) and k(n)
//   count    one CTA per hub: its pin visits by partition (shared histogram), bucket offsets
//   scatter  one CTA per hub: the visits (m, e | inbound-dst bit) into their buckets
//   items    one CTA per partition: eta(n, m) = sum c(e) in a 64-bit and inter(n, m) = sum mu(e)
//            in a 32-bit shared accumulator per key (hubs have S1 = sum c(e) >= 2^32 and in_mu up
//            to Delta: no packed 32-bit form fits them), then Eq.6 validity, purge flags, noise
//            and the partition's top-Pi in one sweep of its table; N(n)'s part to the pool
//   finish   one warp per hub: the k(n) partial lists merged (partitions hold disjoint keys, so
//            the merged list is the node's exact top-Pi), N(n)'s segment published
// eta and inter are the plain integer sums of every tier, so results equal them bit for bit. A
// partition whose table overflows (a hash imbalance far beyond the margin) sends its hub to the
// unfused path.
#include "csr_impl.cuh"
#include "fused.cuh"
#include "scan.cuh"

namespace hgp {

constexpr uint32_t kHubPart = 1536;       // target pin visits per partition (keys <= visits)
constexpr uint32_t kHubMaxParts = 4096;   // histogram / cursor entries in shared memory
constexpr uint32_t kHubLog = 12;          // item table: 4096 slots (16 B each: key, inter, eta), <= 2048 keys
constexpr uint32_t kHubThreads = 256;
constexpr uint32_t kHubKT = 128;          // incident edges per tile (count / scatter)

// partition of neighbour m: a mix independent of hash_slot's multiplicative top bits (otherwise a
// partition's keys would crowd one range of its table)
__device__ __forceinline__ uint32_t hub_part(uint32_t m, uint32_t k) {
  uint32_t h = m * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0xC2B2AE3Du;
  h ^= h >> 13;
  return __umulhi(h, k);
}

struct HubJob {
  FusedJob F;                    // level, params, c(e), (size, in_mu); F.pool = the hub pool
  const uint32_t *list;          // hub nodes
  const uint32_t *list_count;
  uint32_t *hk;                  // [list] partitions (0: not a hub here -> unfused list)
  uint64_t *hb;                  // [list] b(n), then (scan) -> vis_off
  uint32_t *hcnt;                // [list] |N(n)| so far (atomic per partition)
  uint32_t *hfail;               // [list] a partition overflowed
  const uint64_t *item_off;      // [list] exclusive scan of hk
  const uint64_t *vis_off;       // [list] exclusive scan of hb: bucket and N(n) region start
  uint32_t *ibase, *ilen, *inode;   // [items] bucket offset (relative to vis_off), length, list index
  uint32_t *bkey, *bval;         // [sum b] buckets: neighbour id, e | (m in dst(e), e in in(n)) << 31
  hgp_cand *pcand;               // [items][pi] partial top-Pi lists
  uint32_t *lu, *lu_count;       // -> unfused path
};

// plan: one warp per listed node
__global__ void k_hub_plan(HubJob H) {
  const FusedJob &F = H.F;
  const ScoreJob &J = F.S;
  const uint32_t lane = lane_id();
  const uint32_t total = *H.list_count;
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < total; i += gridDim.x * (blockDim.x >> 5)) {
    const uint32_t n = H.list[i];
    uint64_t b = 0;
    for (uint64_t k = J.inc_off[n] + lane; k < J.inc_off[n + 1]; k += 32) {
      const uint32_t e = J.inc[k];
      b += J.edge_off[e + 1] - J.edge_off[e] - 1;
    }
    b = warp_sum(b);
    const uint64_t k = (b + kHubPart - 1) / kHubPart;
    if (lane == 0) {
      H.hcnt[i] = 0;
      H.hfail[i] = 0;
      if (k == 0 || k > kHubMaxParts || J.E >= 0x80000000u) {
        H.hk[i] = 0;
        H.hb[i] = 0;
        H.lu[atomicAdd(H.lu_count, 1u)] = n;
      } else {
        H.hk[i] = (uint32_t)k;
        H.hb[i] = b;
      }
    }
  }
}

// count (SCATTER = false) / scatter (true): one CTA per hub, its pin visits in tiles of kHubKT
// incident edges; flat positions over the tile's rows, the row of a position by binary search.
template <bool SCATTER>
__global__ void __launch_bounds__(kHubThreads) k_hub_visit(HubJob H) {
  constexpr uint32_t NW = kHubThreads / 32;
  __shared__ uint32_t s_h[kHubMaxParts];   // histogram, then (scatter) cursors
  __shared__ uint32_t s_rend[kHubKT], s_rbase[kHubKT], s_rdst[kHubKT], s_ras[kHubKT], s_rad[kHubKT];
  __shared__ uint32_t s_w[NW];
  const FusedJob &F = H.F;
  const ScoreJob &J = F.S;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t total = *H.list_count;
  for (uint32_t i = blockIdx.x; i < total; i += gridDim.x) {
    const uint32_t k = H.hk[i];
    if (k == 0) continue;                                         // CTA-uniform
    const uint32_t n = H.list[i];
    const uint64_t it0 = H.item_off[i], vo = H.vis_off[i];
    for (uint32_t r = tid; r < k; r += kHubThreads) s_h[r] = SCATTER ? H.ibase[it0 + r] : 0u;
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    for (uint64_t t0 = i0; t0 < i1; t0 += kHubKT) {
      const uint32_t kt = (uint32_t)min((uint64_t)kHubKT, i1 - t0);
      uint32_t len = 0, ns = 0, as = 0, ad = 0, a = 0;
      if (tid < kt) {
        const uint32_t e = J.inc[t0 + tid];
        const uint64_t ea = J.edge_off[e];
        a = (uint32_t)ea;                                           // P < 2^32 on the fused path
        len = (uint32_t)(J.edge_off[e + 1] - ea);
        ns = J.edge_nsrc[e];
        as = e;
        ad = e | (t0 + tid < iin ? 0x80000000u : 0u);               // m in dst(e), e in in(n)
      }
      const uint32_t incl = warp_incl_scan(len);
      if (lane == 31) s_w[w] = incl;
      __syncthreads();                                              // (also: s_h initialised)
      uint32_t woff = 0, tot = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) { const uint32_t x = s_w[q]; woff += q < w ? x : 0u; tot += x; }
      if (tid < kt) {
        const uint32_t ex = woff + incl - len;
        s_rend[tid] = ex + len;
        s_rbase[tid] = a - ex;
        s_rdst[tid] = ex + ns;
        s_ras[tid] = as;
        s_rad[tid] = ad;
      }
      __syncthreads();
      for (uint32_t f = tid; f < tot; f += kHubThreads) {
        uint32_t lo = 0, hi = kt - 1;                               // first row whose end exceeds f
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_rend[mid] > f) hi = mid; else lo = mid + 1;
        }
        const uint32_t m = __ldg(J.pins + (s_rbase[lo] + f));
        if (m == n) continue;                                       // self-visits are not neighbours
        const uint32_t p = hub_part(m, k);
        if (SCATTER) {
          const uint64_t pos = vo + atomicAdd(&s_h[p], 1u);
          H.bkey[pos] = m;
          H.bval[pos] = f >= s_rdst[lo] ? s_rad[lo] : s_ras[lo];
        } else {
          atomicAdd(&s_h[p], 1u);
        }
      }
      __syncthreads();                                              // rows are rewritten next tile
    }
    if (!SCATTER) {
      // bucket offsets: exclusive scan of the histogram (each thread a run of consecutive parts)
      const uint32_t per = (k + kHubThreads - 1) / kHubThreads, r0 = min(k, tid * per), r1 = min(k, r0 + per);
      uint32_t run = 0;
      for (uint32_t r = r0; r < r1; ++r) run += s_h[r];
      const uint32_t wincl = warp_incl_scan(run);
      if (lane == 31) s_w[w] = wincl;
      __syncthreads();
      uint32_t base = wincl - run;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) base += q < w ? s_w[q] : 0u;
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t c = s_h[r];
        H.ibase[it0 + r] = base;
        H.ilen[it0 + r] = c;
        H.inode[it0 + r] = i;
        base += c;
      }
    }
    __syncthreads();                                                // s_h / s_w reused next hub
  }
}

// items: one CTA per partition (grid-stride over the items). Table: keys u32 | inter u32 | eta u64.
template <int PIMAX>
__global__ void __launch_bounds__(kHubThreads) k_hub_items(HubJob H, uint32_t nitems) {
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr uint32_t NW = kHubThreads / 32, S = 1u << kHubLog, ucap = S / 2, hmask = S - 1, SW = S / NW;
  __shared__ uint64_t s_tops[(NW + 1) * PIMAX];
  __shared__ uint32_t s_topi[(NW + 1) * PIMAX];
  __shared__ uint32_t s_wsum[NW];
  __shared__ uint32_t s_full;
  __shared__ unsigned long long s_start;
  const FusedJob &F = H.F;
  const ScoreJob &J = F.S;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t *keys = reinterpret_cast<uint32_t *>(dyn);
  uint32_t *inter = keys + S;
  unsigned long long *eta = reinterpret_cast<unsigned long long *>(inter + S);
  const uint32_t keys_s = opaque_u32(smem_u32addr(keys));
  for (uint32_t j = tid; j < S; j += kHubThreads) { keys[j] = kEmpty; inter[j] = 0; eta[j] = 0; }
  if (tid == 0) s_full = 0;
  __syncthreads();
  const uint32_t om32 = J.omega >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)J.omega;
  const uint32_t de32 = J.delta >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)J.delta;
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint32_t i = H.inode[it];
    const uint32_t n = H.list[i];
    const uint64_t base = H.vis_off[i] + H.ibase[it];
    const uint32_t len = H.ilen[it];
    bool full = false;
    for (uint32_t j = tid; j < len; j += kHubThreads) {
      const uint32_t m = H.bkey[base + j], v = H.bval[base + j];
      const uint32_t e = v & 0x7FFFFFFFu;
      uint32_t slot = hash_slot(m, kHubLog), probes = 0;
      while (true) {
        uint32_t kk = lds_u32(keys_s + 4 * slot);
        if (kk == kEmpty) {
          kk = cas_u32(keys_s + 4 * slot, kEmpty, m);
          if (kk == kEmpty) kk = m;
        }
        if (kk == m) {
          atomicAdd(&eta[slot], (unsigned long long)F.cv[e]);    // Eq.5 term c(e)
          if (v >> 31) atomicAdd(&inter[slot], J.edge_mu[e]);     // m in dst(e), e in in(n)
          break;
        }
        if (++probes > kProbeCap) { full = true; break; }
        slot = (slot + 1) & hmask;
      }
    }
    if (full) s_full = 1;
    __syncthreads();
    // occupied slots (n is never inserted): warp w owns [w SW, (w+1) SW)
    uint32_t c1 = 0;
    for (uint32_t j = w * SW + lane; j < (w + 1) * SW; j += 32) c1 += keys[j] != kEmpty;
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c1);
    if (lane == 0) s_wsum[w] = wc;
    __syncthreads();
    uint32_t woff = 0, count = 0;
#pragma unroll
    for (uint32_t q = 0; q < NW; ++q) { const uint32_t x = s_wsum[q]; woff += q < w ? x : 0u; count += x; }
    const bool over = s_full || count > ucap;
    if (tid == 0 && over) H.hfail[i] = 1;
    if (tid == 0 && !over) s_start = H.vis_off[i] + atomicAdd(&H.hcnt[i], count);
    __syncthreads();
    // one sweep: Eq.6 validity, purge flag, noise, top-Pi; clear
    Top<PIMAX> top;
#pragma unroll
    for (int q = 0; q < PIMAX; ++q) { top.s[q] = 0; top.id[q] = 0; }
    const uint32_t wn = J.node_w[n], inn = J.in_mu[n];
    const uint64_t st0 = s_start;
    uint32_t pos = woff;
    for (uint32_t j = w * SW + lane; j < (w + 1) * SW; j += 32) {
      const uint32_t m = keys[j];
      const bool occ = m != kEmpty;
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, occ);
      if (occ) {
        if (!over) {
          const uint2 wm = __ldg(F.wmu + m);                       // (size(m), in_mu(m))
          const uint32_t x = inter[j];
          const bool ok = wn + wm.x <= om32 && inn + (wm.y - x) <= de32;   // |in(n) u in(m)|
          F.pool[st0 + pos + __popc(bal & ((1u << lane) - 1))] = ok ? m : (m | kPurge);
          if (ok) {
            uint64_t sc = eta[j];
            if (J.noise_cap) {
              const uint64_t key = ((uint64_t)min(n, m) << 32) | max(n, m);
              sc += __umul64hi(splitmix64(key ^ J.seed_mix), J.noise_cap + 1);
            }
            top_insert<PIMAX>(top, J.pi, sc, m);
          }
        }
        keys[j] = kEmpty; inter[j] = 0; eta[j] = 0;
      }
      pos += __popc(bal);
    }
    if (tid == 0) s_full = 0;
    if (over) { __syncthreads(); continue; }                        // (the table is clean)
    warp_top_merge<PIMAX>(top, J.pi, s_tops + w * PIMAX, s_topi + w * PIMAX);
    __syncthreads();
    if (w == 0) {
      Top<PIMAX> t2;
#pragma unroll
      for (int q = 0; q < PIMAX; ++q) { t2.s[q] = 0; t2.id[q] = 0; }
      for (uint32_t q = lane; q < NW * J.pi; q += 32) top_insert<PIMAX>(t2, J.pi, s_tops[(q / J.pi) * PIMAX + q % J.pi], s_topi[(q / J.pi) * PIMAX + q % J.pi]);
      warp_top_merge<PIMAX>(t2, J.pi, s_tops + NW * PIMAX, s_topi + NW * PIMAX);
      __syncwarp();
      hgp_cand *crow = H.pcand + (uint64_t)it * J.pi;
      for (uint32_t r = lane; r < J.pi; r += 32) {
        hgp_cand cd;
        cd.score = s_tops[NW * PIMAX + r];
        cd.id = cd.score ? s_topi[NW * PIMAX + r] : kNone;
        cd.pad = 0;
        crow[r] = cd;
      }
    }
    __syncthreads();                                                // s_tops reused by the next item
  }
}

// finish: one warp per hub; merged top-Pi of the partial lists, N(n)'s segment published
template <int PIMAX>
__global__ void k_hub_finish(HubJob H) {
  const FusedJob &F = H.F;
  const ScoreJob &J = F.S;
  const uint32_t lane = lane_id();
  const uint32_t total = *H.list_count;
  __shared__ uint64_t s_s[8][PIMAX];
  __shared__ uint32_t s_i[8][PIMAX];
  const uint32_t wl = threadIdx.x >> 5;
  uint32_t done = 0;
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + wl; i < total; i += gridDim.x * (blockDim.x >> 5)) {
    const uint32_t k = H.hk[i];
    if (k == 0) continue;                                           // warp-uniform
    const uint32_t n = H.list[i];
    if (H.hfail[i]) {
      if (lane == 0) H.lu[atomicAdd(H.lu_count, 1u)] = n;
      continue;
    }
    Top<PIMAX> top;
#pragma unroll
    for (int q = 0; q < PIMAX; ++q) { top.s[q] = 0; top.id[q] = 0; }
    const hgp_cand *pc = H.pcand + H.item_off[i] * J.pi;
    for (uint32_t q = lane; q < k * J.pi; q += 32) {
      const hgp_cand cd = pc[q];
      if (cd.score) top_insert<PIMAX>(top, J.pi, cd.score, cd.id);
    }
    warp_top_merge<PIMAX>(top, J.pi, s_s[wl], s_i[wl]);
    __syncwarp();
    for (uint32_t r = lane; r < J.pi; r += 32) {
      hgp_cand cd;
      cd.score = s_s[wl][r];
      cd.id = cd.score ? s_i[wl][r] : kNone;
      cd.pad = 0;
      J.cand[(uint64_t)n * J.pi + r] = cd;
    }
    if (lane == 0) {
      F.cnt[n - J.lo] = H.hcnt[i];
      F.start[n - J.lo] = H.vis_off[i] + F.start_bias;
      ++done;
    }
    __syncwarp();
  }
  if (lane == 0 && done) tier_add(F.tiers, HGP_TIER_FUSED_H, done);
}

// The hub tier over a device list (hcount = host bound of its count). Nodes it does not finish
// are appended to lu / lu_count (device) for the unfused path. F.pool / F.start / F.cnt: the
// fused level's segment view (hub segments go to a pool of their own, start_bias relative to
// F.pool).
template <int PIMAX>
hgp_status hub_tier_t(hgp_ctx *c, const FusedJob &F0, const uint32_t *list, const uint32_t *list_count,
                      uint32_t hcount, uint32_t *lu, uint32_t *lu_count) {
  if (hcount == 0) return HGP_OK;
  hgp_status st = HGP_OK;
  HubJob H{};
  H.F = F0;
  H.list = list; H.list_count = list_count;
  H.hk = scratch_raw<uint32_t>(c, hcount, &st);
  H.hb = scratch_raw<uint64_t>(c, hcount, &st);
  H.hcnt = scratch_raw<uint32_t>(c, hcount, &st);
  H.hfail = scratch_raw<uint32_t>(c, hcount, &st);
  uint64_t *item_off = scratch_raw<uint64_t>(c, (size_t)hcount + 1, &st);
  uint64_t *vis_off = scratch_raw<uint64_t>(c, (size_t)hcount + 1, &st);
  if (st) return st;
  H.item_off = item_off; H.vis_off = vis_off;
  H.lu = lu; H.lu_count = lu_count;
  const uint32_t gw = div_up(hcount, 8) < 16u * c->sm_count ? div_up(hcount, 8) : 16u * c->sm_count;
  // the listed count may be below hcount: entries past it are never read, but the scans cover
  // hcount entries, so clear them first
  HGP_CUDA(cudaMemsetAsync(H.hk, 0, sizeof(uint32_t) * hcount, c->stream));
  HGP_CUDA(cudaMemsetAsync(H.hb, 0, sizeof(uint64_t) * hcount, c->stream));
  HGP_TRY(launch(c, "hub_plan", k_hub_plan, dim3(gw), dim3(256), 0, H));
  uint64_t nitems = 0, nvis = 0;
  HGP_TRY(scan_exclusive(c, InU32{H.hk}, hcount, item_off, &nitems));
  HGP_TRY(scan_exclusive(c, InU64{H.hb}, hcount, vis_off, &nvis));
  if (nitems == 0) return HGP_OK;
  if (nitems > 0xFFFFFFFFull) return set_error(HGP_E_OVERFLOW, "hub tier: too many partitions");
  H.ibase = scratch_raw<uint32_t>(c, nitems, &st);
  H.ilen = scratch_raw<uint32_t>(c, nitems, &st);
  H.inode = scratch_raw<uint32_t>(c, nitems, &st);
  H.bkey = scratch_raw<uint32_t>(c, nvis, &st);
  H.bval = scratch_raw<uint32_t>(c, nvis, &st);
  H.pcand = scratch_raw<hgp_cand>(c, nitems * F0.S.pi, &st);
  uint32_t *hpool = scratch_raw<uint32_t>(c, nvis, &st);
  if (st) return st;
  H.F.pool = hpool;
  H.F.start_bias = F0.start_bias + (uint64_t)(hpool - F0.pool);
  const uint32_t gh = hcount < 4u * c->sm_count ? hcount : 4u * c->sm_count;
  HGP_TRY(launch(c, "hub_count", k_hub_visit<false>, dim3(gh), dim3(kHubThreads), 0, H));
  HGP_TRY(launch(c, "hub_scatter", k_hub_visit<true>, dim3(gh), dim3(kHubThreads), 0, H));
  const size_t smem = (16u << kHubLog);
  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device))
    cudaFuncSetAttribute(k_hub_items<PIMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const uint32_t gi0 = resident_grid(c, k_hub_items<PIMAX>, kHubThreads, smem);
  const uint32_t gi = nitems < gi0 ? (uint32_t)nitems : gi0;
  HGP_TRY(launch(c, "hub_items", k_hub_items<PIMAX>, dim3(gi), dim3(kHubThreads), smem, H, (uint32_t)nitems));
  HGP_TRY(launch(c, "hub_finish", k_hub_finish<PIMAX>, dim3(gw), dim3(256), 0, H));
  return HGP_OK;
}

hgp_status hub_tier(hgp_ctx *c, const FusedJob &F, const uint32_t *list, const uint32_t *list_count, uint32_t hcount,
                    uint32_t *lu, uint32_t *lu_count) {
  if (F.S.pi <= 4) return hub_tier_t<4>(c, F, list, list_count, hcount, lu, lu_count);
  return hub_tier_t<16>(c, F, list, list_count, hcount, lu, lu_count);
}

}  // namespace hgp
