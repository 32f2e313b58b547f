// score_hub.cu — a3 on an existing N(n) (coarse levels) for the
// nodes whose neighbourhood exceeds the first tier (|N(n)| > 2048): the key-partitioned scheme of
// hub.cu with the bins given. A node's unflagged N(n) entries (key, position) and its pin visits
// (m, e | inbound-dst bit) are bucketed by the same hash of the neighbour into k(n) partitions of
// <= kSHPart bins; one CTA per partition puts its bins in a 2048-slot shared table, adds every
// visit that hits a bin (eta in a u64, inter in a u32: exact for any weights; a visit of a purged
// or removed neighbour finds no bin and is dropped, as in the other tiers), then one sweep runs
// Eq.6 validity, sets the purge flag of each invalid bin at its position in N(n),
// adds noise and keeps the partition's top-Pi; a warp per node merges the partial lists. Nodes it
// cannot take (a partition over the table's half, > 4096 partitions, E >= 2^31) go on to the
// existing tiers, whose results on the same flags are identical (flags only mark invalid bins).
#include "csr_impl.cuh"
#include "fused.cuh"
#include "scan.cuh"

namespace hgp {

constexpr uint32_t kSHPart = 768;        // target bins per partition (table 2048 slots, <= 1024 bins)
constexpr uint32_t kSHMaxParts = 4096;
constexpr uint32_t kSHLog = 11;
constexpr uint32_t kSHThreads = 256;
constexpr uint32_t kSHKT = 128;

__device__ __forceinline__ uint32_t sh_part(uint32_t m, uint32_t k) {   // independent of hash_slot
  uint32_t h = m * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0xC2B2AE3Du;
  h ^= h >> 13;
  return __umulhi(h, k);
}

struct SHubJob {
  ScoreJob J;                     // level, N(n) (nb_off or nb_start/nb_len, relative to lo), params, cand
  const uint64_t *cv;             // [E] c(e)
  const uint2 *wmu;               // [N] (size, in_mu)
  const uint32_t *list, *list_count;
  uint32_t *hk;                   // [list] partitions (0: left to the other tiers)
  uint64_t *hbA, *hbB;            // [list] bins, visits
  const uint64_t *item_off, *offA, *offB;
  uint32_t *ibA, *ilA, *ibB, *ilB, *inode;   // [items]
  uint32_t *akey, *apos;          // bins: key, position in N(n)
  uint32_t *bkey, *bval;          // visits: neighbour, e | (m in dst(e), e in in(n)) << 31
  hgp_cand *pcand;                // [items][pi]
  uint32_t *hfail;
  uint32_t *lu, *lu_count;        // -> the other tiers
};

__device__ __forceinline__ void sh_segment(const ScoreJob &J, uint32_t n, uint64_t &b0, uint64_t &b1) {
  if (J.nb_off) { b0 = J.nb_off[n - J.lo]; b1 = J.nb_off[n - J.lo + 1]; }
  else { b0 = J.nb_start[n - J.lo]; b1 = b0 + J.nb_len[n - J.lo]; }
}

__global__ void k_sh_plan(SHubJob H) {
  const ScoreJob &J = H.J;
  const uint32_t lane = lane_id();
  const uint32_t total = *H.list_count;
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < total; i += gridDim.x * (blockDim.x >> 5)) {
    const uint32_t n = H.list[i];
    uint64_t b0, b1;
    sh_segment(J, n, b0, b1);
    uint64_t bins = 0, b = 0;
    for (uint64_t k = b0 + lane; k < b1; k += 32) bins += !(J.nbr[k] & kPurge);
    for (uint64_t k = J.inc_off[n] + lane; k < J.inc_off[n + 1]; k += 32) {
      const uint32_t e = J.inc[k];
      b += J.edge_off[e + 1] - J.edge_off[e] - 1;
    }
    bins = warp_sum(bins);
    b = warp_sum(b);
    const uint64_t k = (bins + kSHPart - 1) / kSHPart;
    if (lane == 0) {
      H.hfail[i] = 0;
      if (k == 0 || k > kSHMaxParts || J.E >= 0x80000000u) {
        H.hk[i] = 0; H.hbA[i] = 0; H.hbB[i] = 0;
        H.lu[atomicAdd(H.lu_count, 1u)] = n;
      } else {
        H.hk[i] = (uint32_t)k; H.hbA[i] = bins; H.hbB[i] = b;
      }
    }
  }
}

// count (SCATTER = false) / scatter (true): one CTA per node; bins from N(n), visits from I(n)
template <bool SCATTER>
__global__ void __launch_bounds__(kSHThreads) k_sh_visit(SHubJob H) {
  constexpr uint32_t NW = kSHThreads / 32;
  __shared__ uint32_t s_a[kSHMaxParts], s_b[kSHMaxParts];
  __shared__ uint32_t s_rend[kSHKT], s_ns[kSHKT], s_e[kSHKT];
  __shared__ uint64_t s_ra[kSHKT];
  __shared__ uint32_t s_w[NW];
  const ScoreJob &J = H.J;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t total = *H.list_count;
  for (uint32_t i = blockIdx.x; i < total; i += gridDim.x) {
    const uint32_t k = H.hk[i];
    if (k == 0) continue;                                         // CTA-uniform
    const uint32_t n = H.list[i];
    const uint64_t it0 = H.item_off[i], oa = H.offA[i], ob = H.offB[i];
    for (uint32_t r = tid; r < k; r += kSHThreads) {
      s_a[r] = SCATTER ? H.ibA[it0 + r] : 0u;
      s_b[r] = SCATTER ? H.ibB[it0 + r] : 0u;
    }
    __syncthreads();
    // bins: the unflagged entries of N(n) with their positions
    uint64_t b0, b1;
    sh_segment(J, n, b0, b1);
    for (uint64_t q = b0 + tid; q < b1; q += kSHThreads) {
      const uint32_t v = J.nbr[q];
      if (v & kPurge) continue;
      const uint32_t p = sh_part(v, k);
      if (SCATTER) {
        const uint64_t pos = oa + atomicAdd(&s_a[p], 1u);
        H.akey[pos] = v;
        H.apos[pos] = (uint32_t)(q - b0);
      } else {
        atomicAdd(&s_a[p], 1u);
      }
    }
    // visits: the pins of I(n) but n, in tiles of kSHKT incident edges (flat positions, row by
    // binary search)
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    for (uint64_t t0 = i0; t0 < i1; t0 += kSHKT) {
      const uint32_t kt = (uint32_t)min((uint64_t)kSHKT, i1 - t0);
      uint32_t len = 0, ns = 0, ev = 0;
      uint64_t a = 0;
      if (tid < kt) {
        const uint32_t e = J.inc[t0 + tid];
        a = J.edge_off[e];
        len = (uint32_t)(J.edge_off[e + 1] - a);
        ns = J.edge_nsrc[e];
        ev = e | (t0 + tid < iin ? 0x80000000u : 0u);
      }
      const uint32_t incl = warp_incl_scan(len);
      if (lane == 31) s_w[w] = incl;
      __syncthreads();
      uint32_t woff = 0, tot = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) { const uint32_t x = s_w[q]; woff += q < w ? x : 0u; tot += x; }
      if (tid < kt) {
        const uint32_t ex = woff + incl - len;
        s_rend[tid] = ex + len;
        s_ra[tid] = a - ex;                                         // pins index = s_ra + flat position
        s_ns[tid] = ex + ns;                                        // flat start of dst(e)
        s_e[tid] = ev;
      }
      __syncthreads();
      for (uint32_t f = tid; f < tot; f += kSHThreads) {
        uint32_t lo = 0, hi = kt - 1;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_rend[mid] > f) hi = mid; else lo = mid + 1;
        }
        const uint32_t m = __ldg(J.pins + (s_ra[lo] + f));
        if (m == n) continue;
        const uint32_t p = sh_part(m, k);
        if (SCATTER) {
          const uint64_t pos = ob + atomicAdd(&s_b[p], 1u);
          H.bkey[pos] = m;
          const uint32_t ev2 = s_e[lo];
          H.bval[pos] = f >= s_ns[lo] ? ev2 : (ev2 & 0x7FFFFFFFu);    // inbound bit only for dst pins
        } else {
          atomicAdd(&s_b[p], 1u);
        }
      }
      __syncthreads();
    }
    if (!SCATTER) {   // bucket offsets: exclusive scans of both histograms
      const uint32_t per = (k + kSHThreads - 1) / kSHThreads, r0 = min(k, tid * per), r1 = min(k, r0 + per);
      uint32_t runA = 0, runB = 0;
      for (uint32_t r = r0; r < r1; ++r) { runA += s_a[r]; runB += s_b[r]; }
      const uint32_t inA = warp_incl_scan(runA);
      if (lane == 31) s_w[w] = inA;
      __syncthreads();
      uint32_t baseA = inA - runA;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) baseA += q < w ? s_w[q] : 0u;
      __syncthreads();
      const uint32_t inB = warp_incl_scan(runB);
      if (lane == 31) s_w[w] = inB;
      __syncthreads();
      uint32_t baseB = inB - runB;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) baseB += q < w ? s_w[q] : 0u;
      for (uint32_t r = r0; r < r1; ++r) {
        H.ibA[it0 + r] = baseA; H.ilA[it0 + r] = s_a[r];
        H.ibB[it0 + r] = baseB; H.ilB[it0 + r] = s_b[r];
        H.inode[it0 + r] = i;
        baseA += s_a[r]; baseB += s_b[r];
      }
    }
    __syncthreads();
  }
}

// items: one CTA per partition. Table: keys u32 | pos u32 | inter u32 | eta u64 (2048 slots).
template <int PIMAX>
__global__ void __launch_bounds__(kSHThreads) k_sh_items(SHubJob H, uint32_t nitems) {
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr uint32_t NW = kSHThreads / 32, S = 1u << kSHLog, hmask = S - 1, SW = S / NW;
  __shared__ uint64_t s_tops[(NW + 1) * PIMAX];
  __shared__ uint32_t s_topi[(NW + 1) * PIMAX];
  const ScoreJob &J = H.J;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t *keys = reinterpret_cast<uint32_t *>(dyn);
  uint32_t *pos = keys + S;
  uint32_t *inter = pos + S;
  unsigned long long *eta = reinterpret_cast<unsigned long long *>(inter + S + (S & 1));
  const uint32_t keys_s = opaque_u32(smem_u32addr(keys));
  for (uint32_t j = tid; j < S; j += kSHThreads) { keys[j] = kEmpty; inter[j] = 0; eta[j] = 0; }
  __syncthreads();
  const uint32_t om32 = J.omega >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)J.omega;
  const uint32_t de32 = J.delta >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)J.delta;
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint32_t i = H.inode[it];
    const uint32_t n = H.list[i];
    const uint32_t la = H.ilA[it], lb = H.ilB[it];
    if (la > S / 2) {                                               // CTA-uniform: over half the table
      if (tid == 0) H.hfail[i] = 1;
      continue;
    }
    const uint64_t ba = H.offA[i] + H.ibA[it], bb = H.offB[i] + H.ibB[it];
    for (uint32_t j = tid; j < la; j += kSHThreads) {               // bins (distinct keys: no duplicates)
      const uint32_t m = H.akey[ba + j];
      uint32_t slot = hash_slot(m, kSHLog);
      while (cas_u32(keys_s + 4 * slot, kEmpty, m) != kEmpty) slot = (slot + 1) & hmask;   // load <= 1/2
      pos[slot] = H.apos[ba + j];
    }
    __syncthreads();
    for (uint32_t j = tid; j < lb; j += kSHThreads) {               // visits that hit a bin
      const uint32_t m = H.bkey[bb + j];
      uint32_t slot = hash_slot(m, kSHLog);
      uint32_t kk = lds_u32(keys_s + 4 * slot);
      while (kk != m && kk != kEmpty) { slot = (slot + 1) & hmask; kk = lds_u32(keys_s + 4 * slot); }
      if (kk != m) continue;                                        // purged or removed neighbour
      const uint32_t v = H.bval[bb + j], e = v & 0x7FFFFFFFu;
      atomicAdd(&eta[slot], (unsigned long long)H.cv[e]);          // Eq.5 term c(e)
      if (v >> 31) atomicAdd(&inter[slot], J.edge_mu[e]);           // m in dst(e), e in in(n)
    }
    __syncthreads();
    Top<PIMAX> top;
#pragma unroll
    for (int q = 0; q < PIMAX; ++q) { top.s[q] = 0; top.id[q] = 0; }
    uint64_t b0, b1;
    sh_segment(J, n, b0, b1);
    const uint32_t wn = J.node_w[n], inn = J.in_mu[n];
    for (uint32_t j = w * SW + lane; j < (w + 1) * SW; j += 32) {
      const uint32_t m = keys[j];
      if (m == kEmpty) continue;
      const uint2 wm = __ldg(H.wmu + m);
      const uint32_t x = inter[j];
      // |in(n) ∪ in(m)| = in_mu(n) + in_mu(m) - inter
      const bool ok = wn + wm.x <= om32 && inn + (wm.y - x) <= de32;
      if (!ok) {
        J.nbr[b0 + pos[j]] = m | kPurge;                            // purge flag
      } else {
        uint64_t sc = eta[j];
        if (J.noise_cap) {
          const uint64_t key = ((uint64_t)min(n, m) << 32) | max(n, m);
          sc += __umul64hi(splitmix64(key ^ J.seed_mix), J.noise_cap + 1);
        }
        top_insert<PIMAX>(top, J.pi, sc, m);
      }
      keys[j] = kEmpty; inter[j] = 0; eta[j] = 0;
    }
    warp_top_merge<PIMAX>(top, J.pi, s_tops + w * PIMAX, s_topi + w * PIMAX);
    __syncthreads();
    if (w == 0) {
      Top<PIMAX> t2;
#pragma unroll
      for (int q = 0; q < PIMAX; ++q) { t2.s[q] = 0; t2.id[q] = 0; }
      for (uint32_t q = lane; q < NW * J.pi; q += 32)
        top_insert<PIMAX>(t2, J.pi, s_tops[(q / J.pi) * PIMAX + q % J.pi], s_topi[(q / J.pi) * PIMAX + q % J.pi]);
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
    __syncthreads();
  }
}

template <int PIMAX>
__global__ void k_sh_finish(SHubJob H) {
  const ScoreJob &J = H.J;
  const uint32_t lane = lane_id();
  const uint32_t total = *H.list_count;
  __shared__ uint64_t s_s[8][PIMAX];
  __shared__ uint32_t s_i[8][PIMAX];
  const uint32_t wl = threadIdx.x >> 5;
  uint32_t done = 0;
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + wl; i < total; i += gridDim.x * (blockDim.x >> 5)) {
    const uint32_t k = H.hk[i];
    if (k == 0) continue;
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
    if (lane == 0) ++done;
    __syncwarp();
  }
  if (lane == 0 && done) tier_add(J.tiers, HGP_TIER_SCORE_HUB, done);
}

template <int PIMAX>
hgp_status score_hub_t(hgp_ctx *c, const ScoreJob &J, const uint64_t *cv, const uint2 *wmu, const uint32_t *list,
                       const uint32_t *list_count, uint32_t hcount, uint32_t *lu, uint32_t *lu_count) {
  hgp_status st = HGP_OK;
  SHubJob H{};
  H.J = J; H.cv = cv; H.wmu = wmu; H.list = list; H.list_count = list_count; H.lu = lu; H.lu_count = lu_count;
  H.hk = scratch_raw<uint32_t>(c, hcount, &st);
  H.hbA = scratch_raw<uint64_t>(c, hcount, &st);
  H.hbB = scratch_raw<uint64_t>(c, hcount, &st);
  H.hfail = scratch_raw<uint32_t>(c, hcount, &st);
  uint64_t *item_off = scratch_raw<uint64_t>(c, (size_t)hcount + 1, &st);
  uint64_t *offA = scratch_raw<uint64_t>(c, (size_t)hcount + 1, &st);
  uint64_t *offB = scratch_raw<uint64_t>(c, (size_t)hcount + 1, &st);
  if (st) return st;
  H.item_off = item_off; H.offA = offA; H.offB = offB;
  HGP_CUDA(cudaMemsetAsync(H.hk, 0, sizeof(uint32_t) * hcount, c->stream));
  HGP_CUDA(cudaMemsetAsync(H.hbA, 0, sizeof(uint64_t) * hcount, c->stream));
  HGP_CUDA(cudaMemsetAsync(H.hbB, 0, sizeof(uint64_t) * hcount, c->stream));
  const uint32_t gw = div_up(hcount, 8) < 16u * c->sm_count ? div_up(hcount, 8) : 16u * c->sm_count;
  HGP_TRY(launch(c, "shub_plan", k_sh_plan, dim3(gw), dim3(256), 0, H));
  uint64_t nitems = 0, nA = 0, nB = 0;
  HGP_TRY(scan_exclusive(c, InU32{H.hk}, hcount, item_off, &nitems));
  HGP_TRY(scan_exclusive(c, InU64{H.hbA}, hcount, offA, &nA));
  HGP_TRY(scan_exclusive(c, InU64{H.hbB}, hcount, offB, &nB));
  if (nitems == 0) return HGP_OK;
  if (nitems > 0xFFFFFFFFull) return set_error(HGP_E_OVERFLOW, "score hub tier: too many partitions");
  H.ibA = scratch_raw<uint32_t>(c, nitems, &st);
  H.ilA = scratch_raw<uint32_t>(c, nitems, &st);
  H.ibB = scratch_raw<uint32_t>(c, nitems, &st);
  H.ilB = scratch_raw<uint32_t>(c, nitems, &st);
  H.inode = scratch_raw<uint32_t>(c, nitems, &st);
  H.akey = scratch_raw<uint32_t>(c, nA ? nA : 1, &st);
  H.apos = scratch_raw<uint32_t>(c, nA ? nA : 1, &st);
  H.bkey = scratch_raw<uint32_t>(c, nB ? nB : 1, &st);
  H.bval = scratch_raw<uint32_t>(c, nB ? nB : 1, &st);
  H.pcand = scratch_raw<hgp_cand>(c, nitems * J.pi, &st);
  if (st) return st;
  const uint32_t gh = hcount < 4u * c->sm_count ? hcount : 4u * c->sm_count;
  HGP_TRY(launch(c, "shub_count", k_sh_visit<false>, dim3(gh), dim3(kSHThreads), 0, H));
  HGP_TRY(launch(c, "shub_scatter", k_sh_visit<true>, dim3(gh), dim3(kSHThreads), 0, H));
  const size_t smem = (20u << kSHLog) + 16;
  static uint64_t attr_dev = 0;
  if (once_per_device(&attr_dev, c->device))
    cudaFuncSetAttribute(k_sh_items<PIMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const uint32_t gi0 = resident_grid(c, k_sh_items<PIMAX>, kSHThreads, smem);
  HGP_TRY(launch(c, "shub_items", k_sh_items<PIMAX>, dim3(nitems < gi0 ? (uint32_t)nitems : gi0), dim3(kSHThreads), smem,
                 H, (uint32_t)nitems));
  HGP_TRY(launch(c, "shub_finish", k_sh_finish<PIMAX>, dim3(gw), dim3(256), 0, H));
  return HGP_OK;
}

template hgp_status score_hub_t<4>(hgp_ctx *, const ScoreJob &, const uint64_t *, const uint2 *, const uint32_t *,
                                   const uint32_t *, uint32_t, uint32_t *, uint32_t *);
template hgp_status score_hub_t<16>(hgp_ctx *, const ScoreJob &, const uint64_t *, const uint2 *, const uint32_t *,
                                    const uint32_t *, uint32_t, uint32_t *, uint32_t *);

}  // namespace hgp
