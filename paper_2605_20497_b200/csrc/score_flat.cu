// score_flat.cu — a3 for levels whose N(n) already exists: the first tier of
// hgp_score_pairs, built like the fused level-0 kernel (level0.cu).
//
// One CTA (256 threads) per node n with |N(n)| <= 2048:
//  phase 0  sum and gcd of c(e) over I(n) (c(e) precomputed per edge); the node runs PACKED
//           ((eta/g) << ib | inter in one u32, one native shared atomic per visit) when that is
//           exact, else SPLIT (u32 eta + a u16 inter in half a u32 word, exact when sum c(e) < 2^32
//           and in_mu(n) < 2^16: the halves never carry into each other), else it goes to
//           the wide tier (64-bit eta) of score.cu.
//  phase 1  the unflagged entries of N(n) are inserted as bins (and their slots recorded in
//           N(n) order); n itself gets a bin so that self-visits need no test.
//  phase 2  per tile of kFT incident edges: edge rows in shared memory, the tile's pins as one flat
//           sequence split evenly over the warps; per pin one load of the home slot and, if it
//           holds the pin, the add(s) in straight-line code; only displaced keys and purged
//           neighbours (absent bins) take the probe loop.
//  phase 3  validity (Eq.6), purge flags written back into N(n), noise, top-Pi with an
//           early-reject threshold; then only the used slots are reset.
// Results are identical to score.cu's k_score (same integer sums, same tie rules).
#include <type_traits>

#include "csr_impl.cuh"
#include "hashset.cuh"
#include "score_common.cuh"

namespace hgp {

constexpr uint32_t kFT = 128;                 // incident edges per tile
constexpr int kFLog = 12, kFThreads = 256;    // 4096 slots, <= 2048 neighbours
constexpr uint32_t kFCap = 1u << (kFLog - 1);

constexpr uint32_t flat_smem() {
  return (4u << kFLog) + ((4u << kFLog) + 16) + ((2u << kFLog) + 16) + 2 * kFCap + kFT * 24u;
}

// Bins live in 2-slot buckets: a key's probe sequence starts at the even slot (hash & ~1), so a
// lookup reads the whole bucket with one LDS.64 and finds the key there unless both slots were
// taken by others (~1% of keys at the loads of this tier, against ~8% of keys displaced from a
// single home slot). A bucket with an empty slot and no match proves the key absent (linear
// probing), so purged neighbours need no probe either.
__device__ __forceinline__ uint32_t bucket_home(uint32_t key) { return hash_slot(key, kFLog) & ~1u; }
__device__ __forceinline__ uint32_t bucket_insert(uint32_t *keys, uint32_t key) {
  constexpr uint32_t mask = (1u << kFLog) - 1;
  uint32_t s = bucket_home(key);
  volatile uint32_t *vk = keys;
  while (true) {
    const uint32_t k = vk[s];
    if (k == key) return s;
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(&keys[s], kEmpty, key);
      if (old == kEmpty || old == key) return s;
    }
    s = (s + 1) & mask;
  }
}

template <int PIMAX>
__global__ void __launch_bounds__(kFThreads, 4) k_score_flat(ScoreJob J, const uint64_t *cv, const uint2 *wmu) {
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr uint32_t NW = kFThreads / 32, S = 1u << kFLog, hmask = S - 1;
  __shared__ uint64_t s_tops[(NW + 1) * PIMAX];
  __shared__ uint32_t s_topi[(NW + 1) * PIMAX];
  __shared__ uint64_t s_sum[NW], s_g[NW];
  __shared__ uint32_t s_wsum[NW];
  __shared__ uint32_t s_self;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t *keys = reinterpret_cast<uint32_t *>(dyn);
  uint32_t *acc = keys + S;                                         // [S + 4]: slot S = trash
  uint32_t *inter = acc + S + 4;                                    // [S/2 + 4] u16 pairs (SPLIT only)
  uint16_t *nslot = reinterpret_cast<uint16_t *>(inter + S / 2 + 4);  // slot of N(n)[i] (kFCap)
  uint4 *rowA = reinterpret_cast<uint4 *>(nslot + kFCap);
  uint2 *rowB = reinterpret_cast<uint2 *>(rowA + kFT);
  const uint32_t keys_s = opaque_u32(smem_u32addr(keys)), acc_s = opaque_u32(smem_u32addr(acc));
  const uint32_t inter_s = opaque_u32(smem_u32addr(inter));
  const uint32_t rowA_s = opaque_u32(smem_u32addr(rowA)), rowB_s = opaque_u32(smem_u32addr(rowB));
  const uint32_t total = J.list_count ? *J.list_count : J.hi - J.lo;
  uint32_t n_nointer = 0, n_packed = 0, n_split = 0;                // tier counters (thread 0)
  for (uint32_t i = tid; i < S; i += kFThreads) { keys[i] = kEmpty; acc[i] = 0; if (i < S / 2) inter[i] = 0; }
  if (tid < 4) { acc[S + tid] = 0; inter[S / 2 + tid] = 0; }
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t n = J.list ? J.list[t] : J.lo + t;
    uint64_t b0, b1;
    if (J.nb_off) { b0 = J.nb_off[n - J.lo]; b1 = J.nb_off[n - J.lo + 1]; }
    else { b0 = J.nb_start[n - J.lo]; b1 = b0 + J.nb_len[n - J.lo]; }
    const uint32_t cnt = (uint32_t)(b1 - b0);
    if (cnt > kFCap) {                                              // larger tier (CTA-uniform)
      if (tid == 0) J.big_list[atomicAdd(J.big_count, 1u)] = n;
      continue;
    }
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    const uint32_t inn = J.in_mu[n];
    // ---- phase 0 (the first tile's edge data stays in registers)
    uint32_t tlen = 0, tns = 0, tmu = 0;
    uint64_t ta = 0, tce = 0;
    if (tid < kFT && i0 + tid < i1) {
      const uint32_t e = J.inc[i0 + tid];
      ta = J.edge_off[e];
      tlen = (uint32_t)(J.edge_off[e + 1] - ta);
      tns = J.edge_nsrc[e];
      tce = cv[e];
      tmu = i0 + tid < iin ? J.edge_mu[e] : 0u;
    }
    // Eq.6's inbound test can only fail if in_mu(n) + in_mu(m) > Delta for some m; when even the
    // level's largest in_mu keeps it true, inter(n, m) is never needed (the test holds whatever
    // its value) and the bins accumulate eta alone: one shared atomic per visit, no gcd.
    const bool nointer = J.delta == HGP_UNBOUNDED ||
                         (J.max_in_mu && (uint64_t)inn + *J.max_in_mu <= J.delta);
    uint64_t sum = tce;
    for (uint64_t k = i0 + kFT + tid; k < i1; k += kFThreads) sum += cv[J.inc[k]];
    sum = warp_sum(sum);
    if (lane == 0) s_sum[w] = sum;
    __syncthreads();   // also: the table is clean
    uint64_t S1 = 0, g = 1;
#pragma unroll
    for (uint32_t q = 0; q < NW; ++q) S1 += s_sum[q];
    uint32_t ib = 0;
    bool packed;
    const uint32_t ib0 = nointer || !inn ? 0 : 32 - __clz(inn);
    if (nointer && S1 < (1ull << 32)) {
      packed = true;                                                 // acc = eta itself
    } else if (ib0 < 32 && S1 + 1 <= (1ull << (32 - ib0))) {
      packed = true;                                                 // g = 1 already fits: no gcd
      ib = ib0;
    } else {
      // gcd of c(e) over I(n): (eta / g) << ib | inter fits 32 bits more often
      uint64_t gg = tce;
      for (uint64_t k = i0 + kFT + tid; k < i1; k += kFThreads) gg = gcd64(gg, cv[J.inc[k]]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t og = __shfl_xor_sync(0xFFFFFFFFu, gg, o);
        if (og != gg) gg = gcd64(gg, og);
      }
      if (lane == 0) s_g[w] = gg;
      __syncthreads();
      g = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) {
        const uint64_t x = s_g[q];
        if (x != g) g = gcd64(g, x);
      }
      if (g == 0) g = 1;
      ib = nointer || !inn ? 0 : 32 - __clz(inn);
      const uint64_t q1 = S1 / g + 1;
      packed = ib >= 32 ? false : q1 <= (1ull << (32 - ib));
    }
    if (!packed && (S1 >= (1ull << 32) || inn >= (1u << 16))) {     // wide tier (CTA-uniform)
      if (tid == 0) J.wide_list[atomicAdd(J.wide_count, 1u)] = n;
      __syncthreads();
      continue;
    }
    if (!packed) { g = 1; ib = 0; }
    if (tid == 0) {
      if (!packed) ++n_split;
      else if (nointer && ib == 0) ++n_nointer;
      else ++n_packed;
    }
    // ---- phase 1: bins
    for (uint32_t i = tid; i < cnt; i += kFThreads) {
      const uint32_t v = J.nbr[b0 + i];
      uint32_t sl = 0xFFFFu;
      if (!(v & kPurge)) sl = bucket_insert(keys, v);
      nslot[i] = (uint16_t)sl;
    }
    if (tid == 0) s_self = bucket_insert(keys, n);                  // self-visits land in n's slot
    // ---- phase 2, tile by tile
    for (uint64_t t0 = i0; t0 < i1; t0 += kFT) {
      const uint32_t kt = (uint32_t)min((uint64_t)kFT, i1 - t0);
      uint32_t len = 0, ns = 0, as = 0, ad = 0;
      uint64_t a = 0;
      if (tid < kt) {
        uint64_t ce = tce;
        uint32_t mu = nointer ? 0u : tmu;
        if (t0 == i0) {
          a = ta; len = tlen; ns = tns;
        } else {
          const uint32_t e = J.inc[t0 + tid];
          a = J.edge_off[e];
          len = (uint32_t)(J.edge_off[e + 1] - a);
          ns = J.edge_nsrc[e];
          ce = cv[e];
          mu = !nointer && t0 + tid < iin ? J.edge_mu[e] : 0u;
        }
        if (packed) {
          as = (uint32_t)((ce == g ? 1ull : g == 1 ? ce : ce / g) << ib);
          ad = as + mu;                                             // m in dst(e), e in in(n)
        } else {
          as = (uint32_t)ce;                                        // eta term
          ad = mu;                                                  // inter term of a dst pin
        }
      }
      const uint32_t incl = warp_incl_scan(len);
      const bool sh = __any_sync(0xFFFFFFFFu, tid < kt && len < 32);   // bit 31: a short row
      if (lane == 31) s_wsum[w] = incl | (sh ? 0x80000000u : 0u);
      __syncthreads();                                              // also orders phase 1's inserts
      uint32_t woff = 0, tot = 0, anyshort = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) {
        const uint32_t x = s_wsum[q] & 0x7FFFFFFFu;
        anyshort |= s_wsum[q] >> 31;
        woff += q < w ? x : 0u; tot += x;
      }
      const bool longrows = anyshort == 0;
      if (tid < kt) {
        const uint32_t ex = woff + incl - len;
        const uint64_t pp = reinterpret_cast<uint64_t>(J.pins + a) - 4ull * ex;   // &pins[a] - ex
        rowA[tid] = make_uint4((uint32_t)pp, (uint32_t)(pp >> 32), ex + ns, as);
        rowB[tid] = make_uint2(ex + len, ad);
      }
      __syncthreads();
      const uint32_t flo = (uint32_t)(((uint64_t)tot * w) / NW), fhi = (uint32_t)(((uint64_t)tot * (w + 1)) / NW);
      uint32_t k = 0;
      {
        const uint32_t f = flo + lane;
        uint32_t lo_ = 0, hi_ = kt - 1;
        while (lo_ < hi_) {
          const uint32_t mid = (lo_ + hi_) >> 1;
          if (rowB[mid].x > f) hi_ = mid; else lo_ = mid + 1;
        }
        k = lo_;
      }
      uint4 ra = rowA[k];
      uint2 rb = rowB[k];
      auto window = [&](uint32_t f0, auto full_tag, auto long_tag, auto packed_tag) {
        constexpr bool FULL = decltype(full_tag)::value, LONG = decltype(long_tag)::value;
        constexpr bool PK = decltype(packed_tag)::value;   // == packed (CTA-uniform)
        uint32_t m[4], add[4], iad[4], sl[4];
        bool val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t f = f0 + u * 32 + lane;
          val[u] = FULL || f < fhi;
          if (LONG) {
            // rows of >= 32 pins: at most one row end between f - 32 and f (predicated advance)
            const uint32_t lim = FULL ? 0xFFFFFFFFu : fhi;
            asm volatile(
                "{\n .reg .pred pa;\n .reg .b32 ad;\n"
                " setp.ge.u32 pa, %7, %4;\n"
                " setp.lt.and.u32 pa, %7, %10, pa;\n"
                " @pa add.u32 %6, %6, 1;\n"
                " @pa mad.lo.u32 ad, %6, 16, %8;\n"
                " @pa ld.shared.v4.u32 {%0, %1, %2, %3}, [ad];\n"
                " @pa mad.lo.u32 ad, %6, 8, %9;\n"
                " @pa ld.shared.v2.u32 {%4, %5}, [ad];\n}"
                : "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(rb.x), "+r"(rb.y), "+r"(k)
                : "r"(f), "r"(rowA_s), "r"(rowB_s), "r"(lim)
                : "memory");
          } else if (val[u]) {
            while (f >= rb.x) { ++k; ra = rowA[k]; rb = rowB[k]; }
          }
          const uint32_t *pf = reinterpret_cast<const uint32_t *>(((uint64_t)ra.y << 32) | ra.x) + f;
          m[u] = val[u] ? __ldg(pf) : kEmpty;
          const bool dst = f >= ra.z;
          add[u] = PK && dst ? rb.y : ra.w;                         // packed term, or split eta
          iad[u] = !PK && dst ? rb.y : 0u;                          // split: inter += mu
        }
        uint2 kb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          sl[u] = bucket_home(m[u]);
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(kb[u].x), "=r"(kb[u].y) : "r"(keys_s + 4 * sl[u]));
        }
        bool anym = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool h0 = kb[u].x == m[u], h1 = kb[u].y == m[u];
          // hit in the bucket, or absent (an empty slot in the bucket and no match): trash slot S
          const bool hit = h0 || h1;
          const bool absent = !hit && (kb[u].x == kEmpty || kb[u].y == kEmpty);
          const uint32_t slot = hit ? sl[u] + (h1 ? 1u : 0u) : S;
          const bool done = val[u] && (hit || absent);
          if (done) {
            red_add_u32(acc_s + 4 * slot, add[u]);
            if (!PK && iad[u]) red_add_u32(inter_s + 4 * (slot >> 1), iad[u] << (16 * (slot & 1)));
          }
          val[u] = val[u] && !done;                                  // val now marks the rest
          anym |= val[u];
        }
        if (__any_sync(0xFFFFFFFFu, anym)) {                        // both bucket slots taken by others
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (!val[u]) continue;
            uint32_t slot = (sl[u] + 1) & hmask, k2 = kb[u].y;
            while (k2 != m[u]) {
              if (k2 == kEmpty) { slot = S; break; }                 // purged neighbour -> trash
              slot = (slot + 1) & hmask;
              k2 = lds_u32(keys_s + 4 * slot);
            }
            red_add_u32(acc_s + 4 * slot, add[u]);
            if (!PK && iad[u]) red_add_u32(inter_s + 4 * (slot >> 1), iad[u] << (16 * (slot & 1)));
          }
        }
      };
      uint32_t f0 = flo;
      auto windows = [&](auto packed_tag) {
        if (longrows) {
          for (; f0 + 128 <= fhi; f0 += 128) window(f0, std::true_type{}, std::true_type{}, packed_tag);
          if (f0 < fhi) window(f0, std::false_type{}, std::true_type{}, packed_tag);
        } else {
          for (; f0 + 128 <= fhi; f0 += 128) window(f0, std::true_type{}, std::false_type{}, packed_tag);
          if (f0 < fhi) window(f0, std::false_type{}, std::false_type{}, packed_tag);
        }
      };
      if (packed) windows(std::true_type{});
      else windows(std::false_type{});
      __syncthreads();                                              // rows are rewritten by the next tile
    }
    if (i1 == i0) __syncthreads();                                  // phase 1's inserts before phase 3
    // ---- phase 3: validity (Eq.6), flags, noise, top-pi
    const bool small = (unsigned __int128)S1 + J.noise_cap < ((unsigned __int128)1 << 32);   // keys (score << 32 | id)
    const uint64_t wn = J.node_w[n];
    const uint32_t imask = ib ? (uint32_t)((1ull << ib) - 1) : 0u;
    // SMALL: (score << 32 | id) u64 keys with a running threshold; else (u64 score, id) lists.
    // Two instantiations, so only one list is live.
    auto phase3 = [&](auto small_tag) {
      constexpr bool SMALL = decltype(small_tag)::value;
      TopK<PIMAX> topk;
      Top<PIMAX> top;
#pragma unroll
      for (int q = 0; q < PIMAX; ++q) {
        if (SMALL) topk.k[q] = 0;
        else { top.s[q] = 0; top.id[q] = 0; }
      }
      uint64_t thr = 0;
      // 2 entries per thread in flight: slots, then their (size, in_mu) gathers together; each
      // thread clears the slots it read (no separate reset pass over the list)
      for (uint32_t i0 = tid; i0 < cnt; i0 += 2 * kFThreads) {
        uint32_t sl[2], v[2], x[2], xi[2];
        uint2 wm[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t i = i0 + u * kFThreads;
          sl[u] = i < cnt ? nslot[i] : 0xFFFFu;
          v[u] = kEmpty; x[u] = 0; xi[u] = 0;
          if (sl[u] != 0xFFFFu) {
            v[u] = keys[sl[u]];
            x[u] = acc[sl[u]];
            if (!packed) xi[u] = (inter[sl[u] >> 1] >> (16 * (sl[u] & 1))) & 0xFFFFu;
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) wm[u] = sl[u] != 0xFFFFu ? __ldg(wmu + v[u]) : make_uint2(0u, 0u);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (sl[u] == 0xFFFFu) continue;                           // already purged (or past cnt)
          keys[sl[u]] = kEmpty; acc[sl[u]] = 0; inter[sl[u] >> 1] = 0;   // both halves are ours to clear
          uint64_t e_nm, it;
          if (packed) {
            e_nm = (uint64_t)(ib < 32 ? x[u] >> ib : 0) * g;
            it = x[u] & imask;
          } else {
            e_nm = x[u];
            it = xi[u];
          }
          const uint64_t uni = (uint64_t)inn + wm[u].y - it;        // |in(n) ∪ in(m)|
          const bool ok = wn + wm[u].x <= J.omega && (J.delta == HGP_UNBOUNDED || uni <= J.delta);
          if (!ok) { J.nbr[b0 + i0 + u * kFThreads] = v[u] | kPurge; continue; }
          if (SMALL && ((((e_nm + J.noise_cap) << 32) | v[u]) <= thr)) continue;   // cannot enter the top-pi
          uint64_t sc = e_nm;
          if (J.noise_cap) {
            const uint64_t key = ((uint64_t)min(n, v[u]) << 32) | max(n, v[u]);
            sc += __umul64hi(splitmix64(key ^ J.seed_mix), J.noise_cap + 1);    // uniform in [0, cap]
          }
          if (SMALL) {
            const uint64_t key = (sc << 32) | v[u];
            if (key > thr) {
              topk_insert<PIMAX>(topk, J.pi, key);
#pragma unroll
              for (int q = 0; q < PIMAX; ++q)
                if (q == (int)J.pi - 1) thr = topk.k[q];
            }
          } else {
            top_insert<PIMAX>(top, J.pi, sc, v[u]);
          }
        }
      }
      // ---- phase 4: merges (warps, then warp 0)
      if (SMALL) warp_topk_merge<PIMAX>(topk, J.pi, s_tops + w * PIMAX);
      else warp_top_merge<PIMAX>(top, J.pi, s_tops + w * PIMAX, s_topi + w * PIMAX);
      __syncthreads();
      if (w == 0) {
        if (SMALL) {
          TopK<PIMAX> t2;
#pragma unroll
          for (int q = 0; q < PIMAX; ++q) t2.k[q] = 0;
          for (uint32_t i = lane; i < NW * J.pi; i += 32) topk_insert<PIMAX>(t2, J.pi, s_tops[(i / J.pi) * PIMAX + i % J.pi]);
          warp_topk_merge<PIMAX>(t2, J.pi, s_tops + NW * PIMAX);
          __syncwarp();
          for (uint32_t r = lane; r < J.pi; r += 32) {
            const uint64_t kx = s_tops[NW * PIMAX + r];
            hgp_cand cd;
            cd.score = kx >> 32;
            cd.id = kx ? (uint32_t)kx : kNone;
            cd.pad = 0;
            J.cand[(uint64_t)n * J.pi + r] = cd;
          }
        } else {
          Top<PIMAX> t2;
#pragma unroll
          for (int q = 0; q < PIMAX; ++q) { t2.s[q] = 0; t2.id[q] = 0; }
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
      }
    };
    if (small) phase3(std::true_type{});
    else phase3(std::false_type{});
    __syncthreads();
    // (the listed slots were cleared by the threads that read them)
    if (tid == 0) { keys[s_self] = kEmpty; acc[s_self] = 0; inter[s_self >> 1] = 0; acc[S] = 0; inter[S / 2] = 0; }
  }
  if (tid == 0) {
    tier_add(J.tiers, HGP_TIER_SCORE_NOINTER, n_nointer);
    tier_add(J.tiers, HGP_TIER_SCORE_PACKED, n_packed);
    tier_add(J.tiers, HGP_TIER_SCORE_SPLIT, n_split);
  }
}

__global__ void k_pack_wmu2(const uint32_t *node_w, const uint32_t *in_mu, uint32_t N, uint2 *wmu,
                            unsigned int *max_in_mu) {
  uint32_t mx = 0;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    wmu[n] = make_uint2(node_w[n], in_mu[n]);
    mx = max(mx, in_mu[n]);
  }
  mx = warp_max(mx);
  if (lane_id() == 0) atomicMax(max_in_mu, mx);
}

__global__ void k_edge_cv2(const uint64_t *edge_off, const uint32_t *edge_w, uint32_t E, uint32_t norm, uint64_t *cv) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint64_t we = (uint64_t)edge_w[e] << HGP_FP_SHIFT;   // Eq.5 term c(e), 2^-24 fixed point
    cv[e] = norm ? we : we / (edge_off[e + 1] - edge_off[e]);
  }
}

// First tier of a3 on an existing N(n): nodes of the list (or all of [J.lo, J.hi)) with
// |N(n)| <= 2048; larger neighbourhoods -> big_list, nodes needing 64-bit eta -> wide_list.
template <int PIMAX>
hgp_status launch_score_flat(hgp_ctx *c, ScoreJob J, uint32_t nn, uint32_t E, const uint64_t **cv_out,
                             const uint2 **wmu_out) {
  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_score_flat<PIMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, flat_smem());
  }
  hgp_status st = HGP_OK;
  uint64_t *cv = scratch_raw<uint64_t>(c, E ? E : 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "edge_cv", k_edge_cv2, dim3(E ? (div_up(E, 256) < 4096 ? div_up(E, 256) : 4096) : 0), dim3(256), 0,
                 J.edge_off, J.edge_w, E, J.norm, cv));
  uint2 *wmu = scratch_raw<uint2>(c, J.N ? J.N : 1, &st);
  unsigned int *mx = scratch_zero<unsigned int>(c, 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "pack_wmu", k_pack_wmu2, dim3(J.N ? (div_up(J.N, 256) < 4096 ? div_up(J.N, 256) : 4096) : 0), dim3(256),
                 0, J.node_w, J.in_mu, J.N, wmu, mx));
  J.max_in_mu = mx;
  if (cv_out) *cv_out = cv;
  if (wmu_out) *wmu_out = wmu;
  const uint32_t grid = J.list ? 4u * c->sm_count : (nn < 4u * c->sm_count ? (nn ? nn : 1) : 4u * c->sm_count);
  return launch(c, "score_F", k_score_flat<PIMAX>, dim3(grid), dim3(kFThreads), flat_smem(), J, (const uint64_t *)cv,
                (const uint2 *)wmu);
}

template hgp_status launch_score_flat<4>(hgp_ctx *, ScoreJob, uint32_t, uint32_t, const uint64_t **, const uint2 **);
template hgp_status launch_score_flat<16>(hgp_ctx *, ScoreJob, uint32_t, uint32_t, const uint64_t **, const uint2 **);

}  // namespace hgp
