// level0.cu — fused a2 + a3 for the first level, and hgp_coarsen_level0.
//
// At level 0 no neighbour carries a purge flag yet, so materialising N(n) (a2) and
// building the histogram over it (a3) need the same single traversal of I(n) and its
// pins: one CTA per node inserts every pin it meets into a shared-memory hash table (the set
// N(n) ∪ {n}) and, in the same step, adds the pin's packed (c(e)/g << ib | mu-if-inbound) term to
// the slot (native 32-bit shared atomics). Validity, flags, noise and top-Pi then run over the
// node's unique keys, which are also appended (flags included) to N(n). This replaces two
// traversals of the T = sum_e |e|(|e|-1) pin visits by one; results are identical to
// hgp_unique_neighbors followed by hgp_score_pairs (same integer sums, same tie rules).
// Nodes the packed form cannot represent, or whose neighbourhood overflows the largest shared
// table, are handled by the unfused kernels (list mode, over the same segment view).
#include <cstdlib>
#include <type_traits>

#include "csr_impl.cuh"
#include "hashset.cuh"
#include "scan.cuh"
#include "score_common.cuh"
#include "fused.cuh"
#include "pack.cuh"

namespace hgp {

// Shared-memory layout of k_nbrscore: keys[S] | acc[S] | dense (key, acc) pairs uint2[S/2] | rows
// of the current tile of incident edges: uint4 {flat end, pins index - flat start (mod 2^32),
// flat start of dst(e), add of a src pin} and u32 {add of a dst pin}.
constexpr uint32_t kKT = 128;     // incident edges per tile
constexpr uint32_t fused_smem(uint32_t lg) { return (12u << lg) + kKT * 20u; }
constexpr uint32_t fused_smem_list(uint32_t lg) { return (9u << lg) + (lg >= 13 ? 64u : kKT) * 20u; }   // keys, acc, u16 list

// predicated shared CAS: lanes with p == false return `dflt` without touching memory
__device__ __forceinline__ uint32_t cas_u32_if(bool p, uint32_t a, uint32_t cmp, uint32_t val, uint32_t dflt) {
  uint32_t old = dflt;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n @q atom.shared.cas.b32 %0, [%1], %2, %3;\n}"
               : "+r"(old)
               : "r"(a), "r"(cmp), "r"(val), "r"((uint32_t)p)
               : "memory");
  return old;
}

// One CTA per node n (grid-stride over the node list): the fused a2 + a3 traversal of I(n).
//  prologue  the first tile's edge data in registers; one barrier-reduction (__syncthreads_or)
//            tells whether every c(e) over I(n) equals the first one (the common case: then
//            g = c(e), S1/g = |I(n)|, no gcd and no division); otherwise sum and gcd by a block
//            reduction. Is the packed 32-bit accumulator (eta/g << ib | inter) exact?
//  phase 1   per tile of kKT incident edges: edge rows in shared memory (block scan of |e|), then
//            the tile's pins are one flat sequence split evenly over the warps (no idle lanes
//            whatever |e|; each lane tracks its current edge). Per pin, straight-line: one
//            shared load of the home slot and, if it holds the pin (the ~(1 - V/T) of visits
//            that are repeats), one predicated native shared atomic add of the packed term.
//            The rest (first visits: claim an empty slot by CAS and append it to the dense slot
//            list; collision-displaced keys: linear probing) runs once per 128-pin window only
//            if some lane of the warp needs it.
//  phase 2   validity, purge flags, noise and top-Pi over the dense slot list; N(n) to the pool.
//  reset     only the slots used (the table is cleared once per CTA).
// Requires P < 2^32 (32-bit pin indices; the caller routes larger levels to the unfused path).
// LIST (power-law inputs, routed by b(n)): every newly claimed slot is appended to a slot list
// (one warp-aggregated shared atomic per window with claims), so phase 2 reads and clears just the
// node's slots — no sweeps over the S-slot table and no dense array (M's table then fits 3 CTAs
// per SM). Worth it when most visits are first visits (V ~ T); the sweep form is kept for the
// SNN-like inputs where a key is visited ~10 times and claims are rare.
template <int THREADS, int PIMAX, int MINB, int LOG2S, bool LIST = false>
__global__ void __launch_bounds__(THREADS, MINB) k_nbrscore(FusedJob F) {
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr uint32_t NW = THREADS / 32;
  // incident edges per tile: 64 in M's LIST form (its 74.5 KB then fits 3 CTAs per SM, with the
  // 1 KB per-CTA reservation), kKT elsewhere
  constexpr uint32_t KT = (LIST && LOG2S >= 13) ? 64u : kKT;
  static_assert(THREADS >= (int)KT, "one edge row per thread");
  __shared__ uint64_t s_tops[(NW + 1) * PIMAX];
  __shared__ uint32_t s_topi[(NW + 1) * PIMAX];
  __shared__ uint64_t s_sum[NW], s_g[NW];
  __shared__ uint32_t s_wsum[NW];
  __shared__ uint32_t s_full, s_defer, s_n;
  __shared__ unsigned long long s_start;
  const ScoreJob &J = F.S;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr uint32_t S = 1u << LOG2S, ucap = S / 2, hmask = S - 1;
  uint32_t *keys = reinterpret_cast<uint32_t *>(dyn);
  uint32_t *acc = keys + S;
  uint2 *dense = reinterpret_cast<uint2 *>(acc + S);               // (sweep form)
  uint16_t *slist = reinterpret_cast<uint16_t *>(acc + S);         // (LIST: ucap slots)
  static_assert(!LIST || S <= 65536, "u16 slot list");
  uint4 *rows = LIST ? reinterpret_cast<uint4 *>(slist + S / 2) : reinterpret_cast<uint4 *>(dense + S / 2);
  uint32_t *rowd = reinterpret_cast<uint32_t *>(rows + KT);
  // shared-window addresses kept in registers (no rematerialisation inside the pin loop)
  const uint32_t keys_s = opaque_u32(smem_u32addr(keys)), acc_s = keys_s + 4 * S;
  const uint32_t rows_s = opaque_u32(smem_u32addr(rows)), rowd_s = rows_s + 16 * KT;
  const uint32_t total = F.list_count ? *F.list_count : J.hi - J.lo;
  const bool unb = J.delta == HGP_UNBOUNDED;
  const uint64_t mxin = J.max_in_mu ? *J.max_in_mu : 0xFFFFFFFFull;   // max in_mu of the level
  for (uint32_t i = tid; i < S / 4; i += THREADS) {
    reinterpret_cast<uint4 *>(keys)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    reinterpret_cast<uint4 *>(acc)[i] = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) { s_full = 0; s_n = 0; }
  uint32_t done = 0;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t n = F.list ? F.list[t] : J.lo + t;
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    const uint64_t deg = i1 - i0;
    const uint32_t inn = J.in_mu[n];
    // Eq.6's inbound test cannot fail for n when even the level's largest in_mu keeps it true
    // (in_mu(n) + max in_mu <= Delta): then inter(n, m) is never needed — ib = 0, no mu terms,
    // and with a uniform c(e) every pin visit adds exactly 1 (the ADD1 pin loop)
    const bool noint = unb || (uint64_t)inn + mxin <= J.delta;
    // ---- prologue: the first tile's edge data stays in registers
    const bool mine = tid < KT && i0 + tid < i1;
    uint32_t tlen = 0, tns = 0, tmu = 0;
    uint64_t ta = 0, tce = 0;
    if (mine) {
      const uint32_t te = J.inc[i0 + tid];
      ta = J.edge_off[te];
      tlen = (uint32_t)(J.edge_off[te + 1] - ta);
      tns = J.edge_nsrc[te];
      tce = F.cv[te];
      tmu = !noint && i0 + tid < iin ? J.edge_mu[te] : 0u;
    }
    const uint64_t c0 = deg ? F.cv[J.inc[i0]] : 0;                 // broadcast load
    bool diff = mine && tce != c0;
    uint64_t sum = tce;                                            // S1 = sum of c(e), published with B1
#pragma unroll 1
    for (uint64_t k = i0 + KT + tid; k < i1; k += THREADS) {
      const uint64_t ce = F.cv[J.inc[k]];
      diff |= ce != c0;
      sum += ce;
    }
    sum = warp_sum(sum);
    if (lane == 0) s_sum[w] = sum;
    // tile-0 scan of |e|; does every row of the tile have >= 32 pins (then a lane's next flat
    // position, 32 further on, is at most one row end away)?
    // (bit 31 of a warp's published sum: one of its rows is short; sums stay < 2^29 + 2^24)
    const uint32_t tincl = warp_incl_scan(tlen);
    const bool tshort = __any_sync(0xFFFFFFFFu, mine && tlen < 32);
    if (lane == 31) s_wsum[w] = tincl | (tshort ? 0x80000000u : 0u);
    const bool nonuni = __syncthreads_or(diff) != 0;               // B1 (also: the table is clean)
    uint64_t g, S1g;                                               // gcd of c(e), S1 / g
    bool small;                                                    // S1 + cap < 2^32
    if (!nonuni) {
      g = c0 ? c0 : 1;
      S1g = deg;
      small = (unsigned __int128)c0 * deg + J.noise_cap < ((unsigned __int128)1 << 32);
    } else {   // mixed edge sizes or weights (power-law inputs: most nodes)
      // S1 (published with B1); the gcd (a binary-GCD reduction: thousands of instructions per
      // node, measured to dominate small power-law nodes) only when g = 1 leaves the packed form
      // inexact
      uint64_t S1 = 0;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) S1 += s_sum[q];
      const uint32_t ib0 = inn && !noint ? 32 - __clz(inn) : 0;
      g = 1;
      if ((((unsigned __int128)(S1 + 1)) << ib0) > ((unsigned __int128)1 << 32)) {
        uint64_t gg = tce;
#pragma unroll 1
        for (uint64_t k = i0 + KT + tid; k < i1; k += THREADS) gg = gcd64(gg, F.cv[J.inc[k]]);
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
      }
      S1g = g == 1 ? S1 : S1 / g;
      small = (unsigned __int128)S1 + J.noise_cap < ((unsigned __int128)1 << 32);
    }
    const uint32_t ib = inn && !noint ? 32 - __clz(inn) : 0;
    const bool add1 = noint && !nonuni;                            // every visit adds 1
    if ((((unsigned __int128)(S1g + 1)) << ib) > ((unsigned __int128)1 << 32)) {   // packed form inexact
      if (tid == 0) F.defer_list[atomicAdd(F.defer_count, 1u)] = n;
      continue;                                                    // nothing was inserted
    }
    if (tid == 0) keys[hash_slot(n, LOG2S)] = n;                  // the table is clean: n's home; self-visits land there
    // ---- phase 1, tile by tile
    bool full = false;
    for (uint64_t t0 = i0; t0 < i1; t0 += KT) {
      const uint32_t kt = (uint32_t)min((uint64_t)KT, i1 - t0);
      uint32_t len = tlen, ns = tns, mu = tmu, incl = tincl;
      uint64_t a = ta, ce = tce;
      if (t0 != i0) {
        len = 0; ns = 0; mu = 0; a = 0; ce = 0;
        if (tid < kt) {
          const uint32_t e = J.inc[t0 + tid];
          a = J.edge_off[e];
          len = (uint32_t)(J.edge_off[e + 1] - a);
          ns = J.edge_nsrc[e];
          ce = F.cv[e];
          mu = !noint && t0 + tid < iin ? J.edge_mu[e] : 0u;
        }
        incl = warp_incl_scan(len);
        const bool sh = __any_sync(0xFFFFFFFFu, tid < kt && len < 32);
        if (lane == 31) s_wsum[w] = incl | (sh ? 0x80000000u : 0u);
        __syncthreads();
      }
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
        const uint32_t as = (uint32_t)((!nonuni || ce == g ? 1ull : g == 1 ? ce : ce / g) << ib);
        rows[tid] = make_uint4(ex + len, (uint32_t)a - ex, ex + ns, as);
        rowd[tid] = as + mu;                                       // m in dst(e), e in in(n)
      }
      __syncthreads();                                             // B2: rows (and n's slot) visible
      // insert-or-find 4 pins per lane in the table and add their packed terms. FULL: every lane's
      // 4 pins are valid. Claim an empty home (CAS; a first visit); hit if the home now holds m;
      // add the packed term (a miss adds 0 to the slot it looked at: no branch); collision-displaced
      // keys (rare) probe on.
      auto insert4 = [&](const uint32_t (&m)[4], const uint32_t (&add)[4], const bool (&val)[4], auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        uint32_t sl[4], kk[4], miss = 0, clm = 0;                  // clm (LIST): slots claimed, per u
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          sl[u] = hash_slot(m[u], LOG2S);
          kk[u] = lds_u32(keys_s + 4 * sl[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          // claim an empty home (CAS; a first visit); hit if the home now holds m; add the packed
          // term — a miss adds 0 to the slot it looked at (no branch); else report a miss
          uint32_t ms, cl = 0;
          if (LIST && FULL) {
            asm volatile(
                "{\n .reg .pred pc, ph, pk;\n .reg .b32 o;\n"
                " setp.eq.u32 pc, %3, -1;\n"
                " mov.b32 o, %3;\n"
                " @pc atom.shared.cas.b32 o, [%2], -1, %4;\n"
                " setp.eq.u32 pk, o, -1;\n"                          // o == -1 only if the CAS claimed
                " setp.eq.u32 ph, o, %4;\n"
                " or.pred ph, ph, pk;\n"
                " selp.u32 o, %5, 0, ph;\n"
                " red.shared.add.u32 [%2+%6], o;\n"
                " selp.u32 %0, 0, 1, ph;\n"
                " selp.u32 %1, 1, 0, pk;\n}"
                : "=r"(ms), "=r"(cl)
                : "r"(keys_s + 4 * sl[u]), "r"(kk[u]), "r"(m[u]), "r"(add[u]), "n"(4 * S)
                : "memory");
          } else if (LIST) {
            asm volatile(
                "{\n .reg .pred pv, pc, ph, pk;\n .reg .b32 o;\n"
                " setp.ne.u32 pv, %3, 0;\n"
                " setp.eq.and.u32 pc, %4, -1, pv;\n"
                " mov.b32 o, %4;\n"
                " @pc atom.shared.cas.b32 o, [%2], -1, %5;\n"
                " setp.eq.and.u32 pk, o, -1, pv;\n"
                " setp.eq.u32 ph, o, %5;\n"
                " or.pred ph, ph, pk;\n"
                " and.pred ph, ph, pv;\n"
                " selp.u32 o, %6, 0, ph;\n"
                " red.shared.add.u32 [%2+%7], o;\n"
                " not.pred ph, ph;\n"
                " and.pred ph, ph, pv;\n"
                " selp.u32 %0, 1, 0, ph;\n"
                " selp.u32 %1, 1, 0, pk;\n}"
                : "=r"(ms), "=r"(cl)
                : "r"(keys_s + 4 * sl[u]), "r"((uint32_t)val[u]), "r"(kk[u]), "r"(m[u]), "r"(add[u]), "n"(4 * S)
                : "memory");
          } else if (FULL) {
            asm volatile(
                "{\n .reg .pred pc, ph;\n .reg .b32 o;\n"
                " setp.eq.u32 pc, %2, -1;\n"
                " mov.b32 o, %2;\n"
                " @pc atom.shared.cas.b32 o, [%1], -1, %3;\n"
                " setp.eq.u32 ph, o, %3;\n"
                " setp.eq.or.u32 ph, o, -1, ph;\n"
                " selp.u32 o, %4, 0, ph;\n"
                " red.shared.add.u32 [%1+%5], o;\n"
                " selp.u32 %0, 0, 1, ph;\n}"
                : "=r"(ms)
                : "r"(keys_s + 4 * sl[u]), "r"(kk[u]), "r"(m[u]), "r"(add[u]), "n"(4 * S)
                : "memory");
          } else {
            asm volatile(
                "{\n .reg .pred pv, pc, ph;\n .reg .b32 o;\n"
                " setp.ne.u32 pv, %2, 0;\n"
                " setp.eq.and.u32 pc, %3, -1, pv;\n"
                " mov.b32 o, %3;\n"
                " @pc atom.shared.cas.b32 o, [%1], -1, %4;\n"
                " setp.eq.u32 ph, o, %4;\n"
                " setp.eq.or.u32 ph, o, -1, ph;\n"
                " and.pred ph, ph, pv;\n"
                " selp.u32 o, %5, 0, ph;\n"
                " red.shared.add.u32 [%1+%6], o;\n"
                " not.pred ph, ph;\n"
                " and.pred ph, ph, pv;\n"
                " selp.u32 %0, 1, 0, ph;\n}"
                : "=r"(ms)
                : "r"(keys_s + 4 * sl[u]), "r"((uint32_t)val[u]), "r"(kk[u]), "r"(m[u]), "r"(add[u]), "n"(4 * S)
                : "memory");
          }
          miss |= ms << u;
          clm |= cl << u;
        }
        if (__any_sync(0xFFFFFFFFu, miss != 0)) {                  // collision-displaced keys: probe on
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (!((miss >> u) & 1u)) continue;
            uint32_t slot = sl[u], probes = 0, k2;
            bool ok = true;
#pragma unroll 1
            do {
              if (++probes > kProbeCap) { ok = false; break; }
              slot = (slot + 1) & hmask;
              k2 = lds_u32(keys_s + 4 * slot);
              if (k2 == kEmpty) {
                k2 = cas_u32(keys_s + 4 * slot, kEmpty, m[u]);
                if (k2 == kEmpty) {
                  if (LIST) { clm |= 1u << u; sl[u] = slot; }         // claimed further on
                  break;
                }
              }
            } while (k2 != m[u]);
            if (ok) red_add_u32(acc_s + 4 * slot, add[u]);
            else full = true;
          }
        }
        if (LIST && __any_sync(0xFFFFFFFFu, clm != 0)) {            // append the claimed slots
          const uint32_t c = __popc(clm);
          const uint32_t incl = warp_incl_scan(c);
          uint32_t base = 0;
          if (lane == 31 && incl) base = atomicAdd(&s_n, incl);    // lane 31's inclusive sum: the warp's
          base = __shfl_sync(0xFFFFFFFFu, base, 31);
          uint32_t p = base + incl - c;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if ((clm >> u) & 1u) {
              if (p < ucap) slist[p] = (uint16_t)sl[u];
              else full = true;                                  // more keys than the tier holds
              ++p;
            }
          }
        }
      };
      // this warp's share of the tile's flat pin sequence
      const uint32_t flo = (uint32_t)(((uint64_t)tot * w) / NW), fhi = (uint32_t)(((uint64_t)tot * (w + 1)) / NW);
      uint32_t k = 0;
      {
        const uint32_t f = flo + lane;                             // first row whose end exceeds f
        uint32_t lo_ = 0, hi_ = kt - 1;
        while (lo_ < hi_) {
          const uint32_t mid = (lo_ + hi_) >> 1;
          if (rows[mid].x > f) hi_ = mid; else lo_ = mid + 1;
        }
        k = lo_;
      }
      uint4 ra = lds_v4(rows_s + 16 * k);
      uint32_t rd = lds_u32(rowd_s + 4 * k);
      // one 128-pin window of this warp's flat range; FULL: the window lies inside [flo, fhi)
      // ADD1: every visit adds 1 (noint, uniform c(e)): only (row end, pins base) are tracked.
      // fetch: the window's 4 pins per lane (row advance, pin loads); window = fetch + insert4.
      auto fetch = [&](uint32_t f0, uint32_t (&m)[4], uint32_t (&add)[4], bool (&val)[4], auto full_tag, auto long_tag,
                       auto add1_tag) {
        constexpr bool FULL = decltype(full_tag)::value, LONG = decltype(long_tag)::value;
        constexpr bool ADD1 = decltype(add1_tag)::value;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t f = f0 + u * 32 + lane;
          val[u] = FULL || f < fhi;
          if (LONG) {
            // every row has >= 32 pins: at most one row end lies between f - 32 and f, so a
            // predicated single-row advance replaces the loop (no branch); the first position
            // of the warp's range was placed by the binary search
            const uint32_t lim = FULL ? 0xFFFFFFFFu : fhi;
            if (ADD1) {
              asm volatile(
                  "{\n .reg .pred pa;\n .reg .b32 ad;\n"
                  " setp.ge.u32 pa, %3, %0;\n"
                  " setp.lt.and.u32 pa, %3, %4, pa;\n"
                  " @pa add.u32 %2, %2, 1;\n"
                  " @pa mad.lo.u32 ad, %2, 16, %5;\n"
                  " @pa ld.shared.v2.u32 {%0, %1}, [ad];\n}"
                  : "+r"(ra.x), "+r"(ra.y), "+r"(k)
                  : "r"(f), "r"(lim), "r"(rows_s)
                  : "memory");
            } else {
              asm volatile(
                  "{\n .reg .pred pa;\n .reg .b32 ad;\n"
                  " setp.ge.u32 pa, %7, %0;\n"
                  " setp.lt.and.u32 pa, %7, %9, pa;\n"
                  " @pa add.u32 %4, %4, 1;\n"
                  " @pa mad.lo.u32 ad, %4, 16, %6;\n"
                  " @pa ld.shared.v4.u32 {%0, %1, %2, %3}, [ad];\n"
                  " @pa mad.lo.u32 ad, %4, 4, %8;\n"
                  " @pa ld.shared.u32 %5, [ad];\n}"
                  : "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(k), "+r"(rd)
                  : "r"(rows_s), "r"(f), "r"(rowd_s), "r"(lim)
                  : "memory");
            }
          } else if (val[u]) {
            while (f >= ra.x) {                                    // next edge(s)
              ++k;
              if (ADD1) {
                const uint2 r2 = lds_v2(rows_s + 16 * k);
                ra.x = r2.x; ra.y = r2.y;
              } else {
                ra = lds_v4(rows_s + 16 * k);
                rd = lds_u32(rowd_s + 4 * k);
              }
            }
          }
          m[u] = val[u] ? __ldg(J.pins + (ra.y + f)) : 0u;
          add[u] = ADD1 ? 1u : (f >= ra.z ? rd : ra.w);
        }
      };
      auto window = [&](uint32_t f0, auto full_tag, auto long_tag, auto add1_tag) {
        uint32_t m[4], add[4];
        bool val[4];
        fetch(f0, m, add, val, full_tag, long_tag, add1_tag);
        insert4(m, add, val, full_tag);
      };
      uint32_t f0 = flo;
      auto run = [&](auto add1_tag) {
        if (longrows) {
          for (; f0 + 128 <= fhi; f0 += 128) window(f0, std::true_type{}, std::true_type{}, add1_tag);
          if (f0 < fhi) window(f0, std::false_type{}, std::true_type{}, add1_tag);
        } else {
          for (; f0 + 128 <= fhi; f0 += 128) window(f0, std::true_type{}, std::false_type{}, add1_tag);
          if (f0 < fhi) window(f0, std::false_type{}, std::false_type{}, add1_tag);
        }
      };
      if (add1) run(std::true_type{});
      else run(std::false_type{});
      if (full) s_full = 1;
      __syncthreads();                                             // B3: rows are rewritten next
      if (s_full) break;
    }
    if (deg == 0) __syncthreads();                                 // no tile barrier orders n's own key
    if constexpr (LIST) {
      // ---- phase 2 (LIST): the node's keys are the listed slots (n's own home is not listed)
      const uint32_t count = s_n;
      const bool over = s_full != 0;                               // probe cap or list overflow
      if (tid == 0) {
        keys[hash_slot(n, LOG2S)] = kEmpty;                          // n's home (self-visits added there)
        acc[hash_slot(n, LOG2S)] = 0;
        s_defer = 0;
        if (over) {
          F.defer_list[atomicAdd(F.defer_count, 1u)] = n;
        } else {
          const unsigned long long st = atomicAdd(F.pool_cursor, (unsigned long long)count);
          s_start = st;
          F.cnt[n - J.lo] = count;
          if (st + count > F.pool_cap) {
            s_defer = 1;
            F.pool_list[atomicAdd(F.pool_count, 1u)] = n;
          } else {
            F.start[n - J.lo] = st + F.start_bias;
          }
        }
      }
      __syncthreads();                                             // B4: s_start / s_defer; s_n read
      if (tid == 0) { s_full = 0; s_n = 0; }
      if (over) {                                                  // the list may be incomplete: sweep
        for (uint32_t i = tid; i < S / 4; i += THREADS) {
          reinterpret_cast<uint4 *>(keys)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          reinterpret_cast<uint4 *>(acc)[i] = make_uint4(0, 0, 0, 0);
        }
        continue;                                                  // (next node's B1 orders the clear)
      }
      if (s_defer) {
        for (uint32_t i = tid; i < count; i += THREADS) { const uint32_t sl = slist[i]; keys[sl] = kEmpty; acc[sl] = 0; }
        continue;
      }
      if (tid == 0) ++done;
      const ListSrc src{slist, keys_s, acc_s};                     // reads and clears each listed slot
      if (small) eval_packed<PIMAX, THREADS>(J, F, n, count, src, (uint32_t)g, ib, s_start, s_tops, J.cand + (uint64_t)n * J.pi);
      else eval_top<PIMAX, THREADS>(J, F, n, count, src, g, ib, s_start, s_tops, s_topi, J.cand + (uint64_t)n * J.pi);
    } else {
      // ---- phase 2a: count the occupied slots but n's own; warp w owns the slots [w S/NW, (w+1) S/NW),
      //      read 4 per lane (LDS.128)
      constexpr uint32_t SW = S / NW;
      static_assert(SW % 128 == 0, "4 slots per lane per sweep step");
      const uint32_t wbase = w * SW;
      uint32_t c1 = 0;
  #pragma unroll 2
      for (uint32_t j = 4 * lane; j < SW; j += 128) {
        const uint4 k4 = lds_v4(keys_s + 4 * (wbase + j));
        c1 += (uint32_t)(k4.x != kEmpty && k4.x != n) + (uint32_t)(k4.y != kEmpty && k4.y != n) +
              (uint32_t)(k4.z != kEmpty && k4.z != n) + (uint32_t)(k4.w != kEmpty && k4.w != n);
      }
      const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c1);
      if (lane == 0) s_wsum[w] = wc;
      __syncthreads();                                               // B3'
      uint32_t woff = 0, count = 0;
  #pragma unroll
      for (uint32_t q = 0; q < NW; ++q) { const uint32_t x = s_wsum[q]; woff += q < w ? x : 0u; count += x; }
      const bool over = s_full || count > ucap;                      // table too small: next tier
      // ---- phase 2b: pool space for N(n) (thread 0); the warps move the occupied (key, acc) pairs
      //      to the dense array and clear the table behind them (it is clean for the next node)
      if (tid == 0) {
        s_defer = 0;
        if (over) {
          F.defer_list[atomicAdd(F.defer_count, 1u)] = n;
        } else {
          const unsigned long long st = atomicAdd(F.pool_cursor, (unsigned long long)count);
          s_start = st;
          F.cnt[n - J.lo] = count;
          if (st + count > F.pool_cap) {
            s_defer = 1;
            F.pool_list[atomicAdd(F.pool_count, 1u)] = n;
          } else {
            F.start[n - J.lo] = st + F.start_bias;
          }
        }
      }
  #pragma unroll 2
      for (uint32_t j = 4 * lane; j < SW; j += 128) {
        const uint32_t ak = keys_s + 4 * (wbase + j);
        const uint4 k4 = lds_v4(ak);
        const uint4 a4 = lds_v4(ak + 4 * S);
        const bool o0 = k4.x != kEmpty && k4.x != n, o1 = k4.y != kEmpty && k4.y != n;
        const bool o2 = k4.z != kEmpty && k4.z != n, o3 = k4.w != kEmpty && k4.w != n;
        const uint32_t c = (uint32_t)o0 + o1 + o2 + o3;
        const uint32_t incl = warp_incl_scan(c);
        if (!over) {
          uint32_t p = woff + incl - c;
          if (o0) dense[p++] = make_uint2(k4.x, a4.x);
          if (o1) dense[p++] = make_uint2(k4.y, a4.y);
          if (o2) dense[p++] = make_uint2(k4.z, a4.z);
          if (o3) dense[p] = make_uint2(k4.w, a4.w);
        }
        woff += __shfl_sync(0xFFFFFFFFu, incl, 31);
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(ak), "r"(kEmpty) : "memory");
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(ak + 4 * S), "r"(0u) : "memory");
      }
      __syncthreads();                                               // B4
      if (tid == 0) s_full = 0;
      if (over || s_defer) continue;                                 // (the table is already clean)
      if (tid == 0) ++done;
      if (small) eval_packed<PIMAX, THREADS>(J, F, n, count, DenseSrc{dense}, (uint32_t)g, ib, s_start, s_tops, J.cand + (uint64_t)n * J.pi);
      else eval_top<PIMAX, THREADS>(J, F, n, count, DenseSrc{dense}, g, ib, s_start, s_tops, s_topi, J.cand + (uint64_t)n * J.pi);
    }
  }
  if (tid == 0) tier_add(F.tiers, F.tier, done);
}

__global__ void k_pack_wmu(const uint32_t *node_w, const uint32_t *in_mu, uint32_t N, uint2 *wmu,
                           unsigned int *max_in_mu) {
  uint32_t mx = 0;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    wmu[n] = make_uint2(node_w[n], in_mu[n]);
    mx = max(mx, in_mu[n]);
  }
  mx = warp_max(mx);
  if (lane_id() == 0 && mx) atomicMax(max_in_mu, mx);
}

__global__ void k_edge_cv(const uint64_t *edge_off, const uint32_t *edge_w, uint32_t E, uint32_t norm, uint64_t *cv) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint64_t we = (uint64_t)edge_w[e] << HGP_FP_SHIFT;   // Eq.5 term c(e), 2^-24 fixed point
    cv[e] = norm ? we : we / (edge_off[e + 1] - edge_off[e]);
  }
}

__global__ void k_pairs_total(const uint64_t *edge_off, uint32_t E, unsigned long long *T) {
  uint64_t s = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint64_t d = edge_off[e + 1] - edge_off[e];
    s += d * (d - 1);
  }
  s = warp_sum(s);
  if (lane_id() == 0) atomicAdd(T, (unsigned long long)s);
}

__global__ void k_sample_lists(uint32_t lo, uint32_t nn, uint32_t stride, uint32_t *sample, uint32_t *rest,
                               uint32_t *counts) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
    const uint32_t q = i / stride;
    if (i % stride == 0) sample[q] = lo + i;
    else rest[i - q - 1] = lo + i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    counts[0] = (nn + stride - 1) / stride;
    counts[1] = nn - counts[0];
  }
}


// ---------------------------------------------------------------------------------------------
// Tier W: one WARP per small node (bound(n) = sum over I(n) of (|e| - 1) <= kWCap, so at most
// kWCap neighbours): a private 512-slot table per warp, no CTA barriers, no 4096-slot sweeps —
// the per-node fixed costs that dominate power-law inputs (C3/C4: most nodes have ~10-100 pin
// visits) shrink to the warp's own work. Same integer sums and tie rules as the CTA tiers; nodes
// it cannot represent (packed form inexact, scores >= 2^32, a probe run over the cap) are handed
// to the CTA tiers through F.defer_list.
constexpr uint32_t kWLog = 9, kWSlots = 1u << kWLog, kWCap = 256, kWWarps = 8;

// Route by the bound b(n) = sum over I(n) of (|e| - 1) >= |N(n)|: b <= kWCap -> tier W, b <= the
// A table's capacity -> tier A (it cannot overflow), <= B's -> straight to tier M (skipping a
// traversal in A that would only overflow: on power-law inputs nearly every pin visit is a new
// neighbour, so b is close to |N(n)|), larger -> the hub tier (hub.cu).
__global__ void k_small_split(FusedJob F, uint32_t lo, uint32_t nn, uint32_t capA, uint32_t capB, uint32_t *lw,
                              uint32_t *cw, uint32_t *lr, uint32_t *cr, uint32_t *lm, uint32_t *cm, uint32_t *lh,
                              uint32_t *ch) {
  const ScoreJob &J = F.S;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
    const uint32_t n = lo + i;
    uint64_t b = 0;
    for (uint64_t k = J.inc_off[n]; k < J.inc_off[n + 1] && b <= capB; ++k) {
      const uint32_t e = J.inc[k];
      b += J.edge_off[e + 1] - J.edge_off[e] - 1;
    }
    if (b <= kWCap) lw[atomicAdd(cw, 1u)] = n;
    else if (b <= capA) lr[atomicAdd(cr, 1u)] = n;
    else if (b <= capB) lm[atomicAdd(cm, 1u)] = n;
    else lh[atomicAdd(ch, 1u)] = n;                                  // hub: straight to the hub tier
  }
}

template <int PIMAX>
__global__ void __launch_bounds__(kWWarps * 32) k_nbrscore_w(FusedJob F) {
  __shared__ __align__(16) uint32_t s_keys[kWWarps][kWSlots];
  __shared__ __align__(16) uint32_t s_acc[kWWarps][kWSlots];
  const ScoreJob &J = F.S;
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  constexpr uint32_t hmask = kWSlots - 1;
  const uint32_t keys_s = opaque_u32(smem_u32addr(s_keys[w])), acc_s = opaque_u32(smem_u32addr(s_acc[w]));
  uint32_t *keys = s_keys[w], *acc = s_acc[w];
  for (uint32_t i = lane; i < kWSlots; i += 32) { keys[i] = kEmpty; acc[i] = 0; }
  __syncwarp();
  const uint32_t total = *F.list_count;
  uint32_t done = 0;
  for (uint32_t t = blockIdx.x * kWWarps + w; t < total; t += gridDim.x * kWWarps) {
    const uint32_t n = F.list[t];
    const uint64_t i0 = J.inc_off[n], i1 = J.inc_off[n + 1], iin = i0 + J.inc_nin[n];
    const uint32_t inn = J.in_mu[n];
    // sum of c(e) over I(n); the gcd g only if g = 1 leaves the packed accumulator
    // (eta/g << ib | inter) inexact (a binary-GCD reduction costs thousands of instructions)
    uint64_t sum = 0;
    for (uint64_t k = i0 + lane; k < i1; k += 32) sum += F.cv[J.inc[k]];
    sum = warp_sum(sum);
    const uint32_t ib = inn ? 32 - __clz(inn) : 0;
    uint64_t gg = 1;
    if ((((unsigned __int128)(sum + 1)) << ib) > ((unsigned __int128)1 << 32)) {
      gg = 0;
      for (uint64_t k = i0 + lane; k < i1; k += 32) gg = gcd64(gg, F.cv[J.inc[k]]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t og = __shfl_xor_sync(0xFFFFFFFFu, gg, o);
        if (og != gg) gg = gcd64(gg, og);
      }
    }
    const uint64_t g = gg ? gg : 1;
    const bool exact = (((unsigned __int128)(sum / g + 1)) << ib) <= ((unsigned __int128)1 << 32);
    const bool small = (unsigned __int128)sum + J.noise_cap < ((unsigned __int128)1 << 32);
    if (!exact || !small) {
      if (lane == 0) F.defer_list[atomicAdd(F.defer_count, 1u)] = n;
      continue;
    }
    if (lane == 0) keys[hash_slot(n, kWLog)] = n;                 // self-visits land in n's slot
    __syncwarp();
    bool full = false;
    // incident edges 32 at a time (lane = edge), their pins as one flat sequence over the lanes
    for (uint64_t c0 = i0; c0 < i1; c0 += 32) {
      const bool mine = c0 + lane < i1;
      uint32_t len = 0, ns = 0, as = 0, ad = 0, a = 0;
      if (mine) {
        const uint32_t e = J.inc[c0 + lane];
        const uint64_t ea = J.edge_off[e];
        a = (uint32_t)ea;                                          // P < 2^32 on this path
        len = (uint32_t)(J.edge_off[e + 1] - ea);
        ns = J.edge_nsrc[e];
        const uint64_t ce = F.cv[e];
        as = (uint32_t)((ce == g ? 1ull : g == 1 ? ce : ce / g) << ib);
        ad = as + (c0 + lane < iin ? J.edge_mu[e] : 0u);           // m in dst(e), e in in(n)
      }
      const uint32_t incl = warp_incl_scan(len);
      const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
      for (uint32_t f0 = 0; f0 < tot; f0 += 32) {
        const uint32_t f = f0 + lane;
        const bool val = f < tot;
        // the edge holding flat position f: the first lane r with incl[r] > f (5 shuffles)
        uint32_t r = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
          const uint32_t x = __shfl_sync(0xFFFFFFFFu, incl, r + st - 1);
          if (x <= f) r += st;
        }
        const uint32_t rs = __shfl_sync(0xFFFFFFFFu, incl - len, r), ra = __shfl_sync(0xFFFFFFFFu, a, r);
        const uint32_t rns = __shfl_sync(0xFFFFFFFFu, ns, r), ras = __shfl_sync(0xFFFFFFFFu, as, r);
        const uint32_t rad = __shfl_sync(0xFFFFFFFFu, ad, r);
        if (!val) continue;
        const uint32_t j = f - rs;
        const uint32_t m = __ldg(J.pins + ra + j);
        const uint32_t add = j >= rns ? rad : ras;
        uint32_t slot = hash_slot(m, kWLog), probes = 0;
        while (true) {
          uint32_t k = lds_u32(keys_s + 4 * slot);
          if (k == kEmpty) {
            k = cas_u32(keys_s + 4 * slot, kEmpty, m);
            if (k == kEmpty) k = m;
          }
          if (k == m) { red_add_u32(acc_s + 4 * slot, add); break; }
          if (++probes > kProbeCap) { full = true; break; }
          slot = (slot + 1) & hmask;
        }
      }
    }
    __syncwarp();
    if (__any_sync(0xFFFFFFFFu, full)) {                           // (cannot happen below 1/2 load)
      for (uint32_t i = lane; i < kWSlots; i += 32) { keys[i] = kEmpty; acc[i] = 0; }
      __syncwarp();
      if (lane == 0) F.defer_list[atomicAdd(F.defer_count, 1u)] = n;
      continue;
    }
    // the occupied slots but n's: count, reserve N(n) in the pool, validity / flags / noise and the
    // warp's top-Pi over 4 slots per lane per step; the table is cleared behind the sweep
    uint32_t cnt = 0;
#pragma unroll
    for (uint32_t j = 4 * lane; j < kWSlots; j += 128) {
      const uint4 k4 = lds_v4(keys_s + 4 * j);
      cnt += (uint32_t)(k4.x != kEmpty && k4.x != n) + (uint32_t)(k4.y != kEmpty && k4.y != n) +
             (uint32_t)(k4.z != kEmpty && k4.z != n) + (uint32_t)(k4.w != kEmpty && k4.w != n);
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    unsigned long long st0 = 0;
    if (lane == 0) st0 = atomicAdd(F.pool_cursor, (unsigned long long)cnt);
    st0 = __shfl_sync(0xFFFFFFFFu, st0, 0);
    const bool pool_ok = st0 + cnt <= F.pool_cap;
    if (lane == 0) {
      F.cnt[n - J.lo] = cnt;
      if (pool_ok) F.start[n - J.lo] = st0 + F.start_bias;
      else F.pool_list[atomicAdd(F.pool_count, 1u)] = n;
    }
    const EvalCtx E = eval_ctx(J, n, ib);
    const uint32_t g32 = (uint32_t)g, cap32 = (uint32_t)J.noise_cap;
    uint64_t carry = 0;
    uint32_t pos = 0;
#pragma unroll
    for (uint32_t j = 4 * lane; j < kWSlots; j += 128) {
      const uint4 k4 = lds_v4(keys_s + 4 * j);
      const uint4 a4 = lds_v4(acc_s + 4 * j);
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(keys_s + 4 * j), "r"(kEmpty) : "memory");
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(acc_s + 4 * j), "r"(0u) : "memory");
      const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w}, aa[4] = {a4.x, a4.y, a4.z, a4.w};
      bool occ[4];
      uint32_t c = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) { occ[u] = kk[u] != kEmpty && kk[u] != n; c += occ[u]; }
      const uint32_t incl = warp_incl_scan(c);
      uint32_t p = pos + incl - c;
      uint64_t key[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        key[u] = 0;
        if (!occ[u] || !pool_ok) continue;
        uint32_t cn;
        if (eval_one(F, E, make_uint2(kk[u], aa[u]), st0 + p, cn)) {
          uint32_t s32 = cn * g32;                                 // eta(n, m) < 2^32
          if (cap32) {
            const uint64_t hk = ((uint64_t)min(n, kk[u]) << 32) | max(n, kk[u]);
            s32 += (uint32_t)__umul64hi(splitmix64(hk ^ J.seed_mix), J.noise_cap + 1);   // uniform in [0, cap]
          }
          key[u] = ((uint64_t)s32 << 32) | kk[u];
        }
        ++p;
      }
      pos += __shfl_sync(0xFFFFFFFFu, incl, 31);
      uint64_t nc = 0;
      for (uint32_t rr = 0; rr < J.pi; ++rr) {                      // the warp's pi best so far
        uint64_t lm = carry;
#pragma unroll
        for (int u = 0; u < 4; ++u) lm = key[u] > lm ? key[u] : lm;
        const uint32_t hi = (uint32_t)(lm >> 32);
        const uint32_t mhi = __reduce_max_sync(0xFFFFFFFFu, hi);
        if (mhi == 0) break;
        const uint32_t mlo = __reduce_max_sync(0xFFFFFFFFu, hi == mhi ? (uint32_t)lm : 0u);
        const uint64_t K = ((uint64_t)mhi << 32) | mlo;
        if (carry == K) carry = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (key[u] == K) key[u] = 0;
        if (lane == rr) nc = K;
      }
      carry = nc;
    }
    __syncwarp();
    if (pool_ok) {
      for (uint32_t rr = lane; rr < J.pi; rr += 32) {
        hgp_cand cd;
        cd.score = carry >> 32;
        cd.id = carry ? (uint32_t)carry : kNone;
        cd.pad = 0;
        J.cand[(uint64_t)n * J.pi + rr] = cd;
      }
      if (lane == 0) ++done;
    }
  }
  if (lane == 0) tier_add(F.tiers, HGP_TIER_FUSED_W, done);
}

// tiers of the fused kernel: A 4096 slots (40 KB incl. the dense list) for every node, M 8192
// slots (72 KB, 3 CTAs/SM), B 16384 slots (144 KB, 1 CTA/SM); what B cannot hold (or the packed
// accumulator cannot represent) goes to the unfused kernels.
static constexpr int kFALog = 12, kFMLog = 13, kFBLog = 14;
static constexpr uint32_t kFMThreads = 256, kFBThreads = 256;
// A's LIST form (routed power-law nodes, ~1,000 visits each): 4 warps per node, 5 nodes per SM —
// per-node latency (dependent loads, barriers) bounds these nodes, so nodes in flight count more
// than warps per node
static constexpr uint32_t kFALThreads = 128;

struct TierLists {
  const uint32_t *in_list, *in_count;   // nullptr: every node of [lo, hi)
  uint32_t hn;                          // host upper bound of the input count (grid sizing)
  uint32_t *la, *ca, *lm, *cm;          // A -> M, M -> B hand-off
  uint32_t *ld, *cd;                    // B -> unfused (appended)
  bool small_first;                     // route small nodes to tier W first (range input only)
  bool list_mode = false;               // A and M in their LIST form (the routed power-law path)
};


template <int PIMAX, int TA, int MINB>
hgp_status fused_tiers_t(hgp_ctx *c, FusedJob F, const TierLists &L) {
  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_nbrscore<TA, PIMAX, MINB, kFALog>, cudaFuncAttributeMaxDynamicSharedMemorySize, fused_smem(kFALog));
    cudaFuncSetAttribute(k_nbrscore<kFMThreads, PIMAX, 3, kFMLog>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fused_smem(kFMLog));
    cudaFuncSetAttribute(k_nbrscore<kFBThreads, PIMAX, 1, kFBLog>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fused_smem(kFBLog));
    cudaFuncSetAttribute(k_nbrscore<kFALThreads, PIMAX, 5, kFALog, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fused_smem_list(kFALog));
    cudaFuncSetAttribute(k_nbrscore<kFMThreads, PIMAX, 3, kFMLog, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fused_smem_list(kFMLog));
  }
  const uint32_t sm = c->sm_count;
  const uint32_t per_sm = MINB;                                     // exactly the resident CTAs
  const uint32_t gA = L.hn < per_sm * sm ? L.hn : per_sm * sm;
  if (gA == 0) return HGP_OK;
  // M and B: exactly the resident CTAs (M's 98 KB table fits 2 per SM, not its register bound 3)
  const uint32_t gM = resident_grid(c, k_nbrscore<kFMThreads, PIMAX, 3, kFMLog>, kFMThreads, fused_smem(kFMLog));
  const uint32_t gB = resident_grid(c, k_nbrscore<kFBThreads, PIMAX, 1, kFBLog>, kFBThreads, fused_smem(kFBLog));
  if (!L.in_list && L.small_first) {
    // tier W first: nodes with <= kWCap pin visits, one warp each; the rest (and W's deferrals)
    // continue below as a list
    hgp_status st = HGP_OK;
    uint32_t *lw = scratch_raw<uint32_t>(c, L.hn, &st), *lr = scratch_raw<uint32_t>(c, L.hn, &st);
    uint32_t *cnt2 = scratch_zero<uint32_t>(c, 2, &st);
    if (st) return st;
    HGP_TRY(launch(c, "small_split", k_small_split, dim3(div_up(L.hn, 256) < 4096 ? div_up(L.hn, 256) : 4096), dim3(256),
                   0, F, F.S.lo, L.hn, (1u << kFALog) / 2, (1u << kFBLog) / 2, lw, cnt2, lr, cnt2 + 1, L.la, L.ca,
                   L.ld, L.cd));
    FusedJob FW = F;
    FW.list = lw; FW.list_count = cnt2; FW.defer_list = lr; FW.defer_count = cnt2 + 1;
    HGP_TRY(launch(c, "nbrscore_W", k_nbrscore_w<PIMAX>, dim3(16 * sm), dim3(kWWarps * 32), 0, FW));
    TierLists L2 = L;
    L2.in_list = lr; L2.in_count = cnt2 + 1; L2.small_first = false; L2.list_mode = true;
    return fused_tiers_t<PIMAX, TA, MINB>(c, F, L2);
  }
  constexpr uint32_t kStride = 64;
  const uint64_t sample_min = c->opt.fused_sample_min;            // 1024 * kStride by default
  if (!L.in_list && L.hn >= sample_min && L.hn >= 2 * kStride) {
    // Tier A on every 64th node first: if most of them overflow its table (large neighbourhoods,
    // e.g. the rewired SNN), the other nodes start in tier M instead of paying a wasted traversal
    // in A. Results do not depend on the choice (every tier computes the same exact values).
    hgp_status st = HGP_OK;
    uint32_t *sample = scratch_raw<uint32_t>(c, L.hn / kStride + 1, &st);
    uint32_t *rest = scratch_raw<uint32_t>(c, L.hn, &st);
    uint32_t *cnt2 = scratch_zero<uint32_t>(c, 2, &st);
    if (st) return st;
    HGP_TRY(launch(c, "sample_lists", k_sample_lists, dim3(div_up(L.hn, 256) < 4096 ? div_up(L.hn, 256) : 4096), dim3(256),
                   0, F.S.lo, L.hn, kStride, sample, rest, cnt2));
    F.list = sample; F.list_count = cnt2; F.log2s = kFALog; F.tier = HGP_TIER_FUSED_S;
    F.defer_list = L.la; F.defer_count = L.ca;
    HGP_TRY(launch(c, "nbrscore_S", k_nbrscore<TA, PIMAX, MINB, kFALog>, dim3(gA), dim3(TA), fused_smem(kFALog), F));
    uint32_t deferred = 0;
    HGP_TRY(read_back(c, L.ca, 4, &deferred));
    const uint32_t ns = (L.hn + kStride - 1) / kStride;
    F.list = rest; F.list_count = cnt2 + 1;
    F.tier = HGP_TIER_FUSED_A;
    if (4 * deferred > ns) {                                        // > 25 %: start in M
      F.log2s = kFMLog; F.tier = HGP_TIER_FUSED_M; F.defer_list = L.lm; F.defer_count = L.cm;
      HGP_TRY(launch(c, "nbrscore_M", k_nbrscore<kFMThreads, PIMAX, 3, kFMLog>, dim3(gM), dim3(kFMThreads),
                     fused_smem(kFMLog), F));
    } else {
      HGP_TRY(launch(c, "nbrscore_A", k_nbrscore<TA, PIMAX, MINB, kFALog>, dim3(gA), dim3(TA), fused_smem(kFALog), F));
    }
  } else {
    F.list = L.in_list; F.list_count = L.in_count; F.log2s = kFALog; F.tier = HGP_TIER_FUSED_A;
    F.defer_list = L.la; F.defer_count = L.ca;
    if (L.list_mode)
      HGP_TRY(launch(c, "nbrscore_A", k_nbrscore<kFALThreads, PIMAX, 5, kFALog, true>,
                     dim3(std::min(L.hn, resident_grid(c, k_nbrscore<kFALThreads, PIMAX, 5, kFALog, true>, kFALThreads,
                                                        fused_smem_list(kFALog)))),
                     dim3(kFALThreads),
                     fused_smem_list(kFALog), F));
    else
      HGP_TRY(launch(c, "nbrscore_A", k_nbrscore<TA, PIMAX, MINB, kFALog>, dim3(gA), dim3(TA), fused_smem(kFALog), F));
  }
  F.list = L.la; F.list_count = L.ca; F.log2s = kFMLog; F.tier = HGP_TIER_FUSED_M;
  F.defer_list = L.lm; F.defer_count = L.cm;
  if (L.list_mode) {   // 74.5 KB: 3 CTAs per SM (the sweep form's 98.5 KB allows 2)
    const uint32_t gML = resident_grid(c, k_nbrscore<kFMThreads, PIMAX, 3, kFMLog, true>, kFMThreads, fused_smem_list(kFMLog));
    HGP_TRY(launch(c, "nbrscore_M", k_nbrscore<kFMThreads, PIMAX, 3, kFMLog, true>, dim3(gML), dim3(kFMThreads),
                   fused_smem_list(kFMLog), F));
  } else {
    HGP_TRY(launch(c, "nbrscore_M", k_nbrscore<kFMThreads, PIMAX, 3, kFMLog>, dim3(gM), dim3(kFMThreads), fused_smem(kFMLog), F));
  }
  F.list = L.lm; F.list_count = L.cm; F.log2s = kFBLog; F.tier = HGP_TIER_FUSED_B;
  F.defer_list = L.ld; F.defer_count = L.cd;
  HGP_TRY(launch(c, "nbrscore_B", k_nbrscore<kFBThreads, PIMAX, 1, kFBLog>, dim3(gB), dim3(kFBThreads), fused_smem(kFBLog), F));
  return HGP_OK;
}

template <int PIMAX>
hgp_status fused_tiers(hgp_ctx *c, FusedJob F, const TierLists &L) {
  return fused_tiers_t<PIMAX, 256, 4>(c, F, L);   // 64 registers, 4 CTAs/SM (measured faster than 48 / 5)
}

__global__ void k_list_cnt_sum(const uint32_t *list, const uint32_t *count, const uint32_t *cnt, uint32_t lo,
                               unsigned long long *sum) {
  uint64_t s = 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < *count; t += gridDim.x * blockDim.x) s += cnt[list[t] - lo];
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(sum, (unsigned long long)s);
}

__global__ void k_iota(uint32_t *list, uint32_t *count, uint32_t lo, uint32_t nn) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += gridDim.x * blockDim.x) list[t] = lo + t;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = nn;
}

__global__ void k_cnt_sum(const uint32_t *cnt, uint32_t nn, unsigned long long *sum) {
  uint64_t s = 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += gridDim.x * blockDim.x) s += cnt[t];
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(sum, (unsigned long long)s);
}

// a2 + a3 on a level-0 CSR (no flags yet). Returns the same nb and cand as hgp_unique_neighbors
// followed by hgp_score_pairs. Synchronises.
hgp_status nbrs_score_fused(hgp_ctx *c, const hgp_csr *g, const hgp_params *p, uint32_t lo, uint32_t hi,
                            hgp_nbrs *out, hgp_cand *cand, SegView *view) {
  if (out) memset(out, 0, sizeof(*out));
  const uint32_t nn = hi - lo;
  ScoreJob J;
  HGP_TRY(score_prologue(c, g, lo, hi, p, &J));
  J.cand = cand;
  hgp_status st = HGP_OK;
  unsigned long long *misc = scratch_zero<unsigned long long>(c, 4, &st);    // T, cursor, cursor 2, sum
  uint32_t *counts = scratch_zero<uint32_t>(c, 16, &st);
  uint64_t *start = scratch_raw<uint64_t>(c, nn, &st);
  uint32_t *cnt = scratch_raw<uint32_t>(c, nn, &st);
  uint32_t *lists = scratch_raw<uint32_t>(c, 4 * (size_t)(nn ? nn : 1), &st);
  if (st) return st;
  if (nn == 0) return HGP_E_INTERNAL;   // handled by the caller's fallback
  if (g->P >= (1ull << 32)) return HGP_E_INTERNAL;   // the fused kernel indexes pins with 32 bits
  HGP_TRY(launch(c, "pairs_total", k_pairs_total, dim3(g->E ? (div_up(g->E, 256) < 1024 ? div_up(g->E, 256) : 1024) : 0),
                 dim3(256), 0, (const uint64_t *)g->edge_off, g->E, misc));
  uint64_t T = 0;
  HGP_TRY(read_u64(c, (const uint64_t *)misc, &T));
  // pool: T = sum_n b(n) bounds V exactly (|N(n)| <= b(n) = sum over I(n) of (|e| - 1)), scaled to
  // the range. A smaller estimate (24 P was used) sends every node past it through a second, exact
  // pool — a second full traversal: on power-law inputs V ~ T (C3: V = 7.2e9 = 0.95 T, 24 P = 1.2e9)
  // and the level paid both (measured: A+M+B 192 ms then 307 ms again).
  const double frac = g->N ? (double)nn / g->N : 1.0;
  uint64_t pool_cap = (uint64_t)(T * (frac < 1.0 ? 1.25 * frac : 1.0)) + nn;
  // at most 2^34 entries (64 GB; C5's T would be 396 GB); nodes that do not fit go to the exact
  // second pool. (A cap from cudaMemGetInfo was measured to misfire: the caching allocator's
  // reserved blocks read as used, the pool shrank and the level took the slow second-pool path.)
  if (pool_cap > (1ull << 34)) pool_cap = 1ull << 34;
  // test hooks (tests/test_gpu_parity.py, hgp_ctx_set_option): a tiny first pool, or every node
  // on the unfused path
  if (c->opt.fused_pool_cap) pool_cap = c->opt.fused_pool_cap;
  const bool all_unfused = c->opt.unfused;
  if (pool_cap == 0) pool_cap = 1;
  uint32_t *pool = scratch_raw<uint32_t>(c, pool_cap, &st);
  if (st) return st;
  uint32_t *LA = lists, *LM = lists + nn, *LD = lists + 2 * (size_t)nn, *LP = lists + 3 * (size_t)nn;
  // (counts 8: the nodes the hub tier leaves to the unfused path, listed in LA)
  // counts: 0 A->M, 1 M->B, 2 deferred (unfused), 3 pool overflow, 4/5 second pass A->M / M->B,
  // 6 second-pass pool overflow (impossible: exact pool), 7 max degree
  uint64_t *cv = scratch_raw<uint64_t>(c, g->E ? g->E : 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "edge_cv", k_edge_cv, dim3(g->E ? (div_up(g->E, 256) < 4096 ? div_up(g->E, 256) : 4096) : 0), dim3(256), 0,
                 (const uint64_t *)g->edge_off, (const uint32_t *)g->edge_w, g->E, p->norm, cv));
  uint2 *wmu = scratch_raw<uint2>(c, g->N ? g->N : 1, &st);
  unsigned int *mxin = scratch_zero<unsigned int>(c, 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "pack_wmu", k_pack_wmu, dim3(g->N ? (div_up(g->N, 256) < 4096 ? div_up(g->N, 256) : 4096) : 0),
                 dim3(256), 0, (const uint32_t *)g->node_w, (const uint32_t *)g->in_mu, g->N, wmu, mxin));
  J.max_in_mu = mxin;
  FusedJob F{};
  F.S = J;
  F.cv = cv;
  F.wmu = wmu;
  F.tiers = c->d_tiers;
  F.pool = pool; F.pool_cap = pool_cap; F.pool_cursor = misc + 1; F.start = start; F.cnt = cnt;
  F.pool_list = LP; F.pool_count = counts + 3;
  // power-law inputs (few pins per node on average) are mostly small nodes: warp-per-node tier first
  TierLists L{nullptr, nullptr, nn, LA, counts + 0, LM, counts + 1, LD, counts + 2, g->P <= 32ull * g->N};
  if (all_unfused) HGP_TRY(launch(c, "iota", k_iota, dim3(div_up(nn, 256) < 4096 ? div_up(nn, 256) : 4096), dim3(256), 0,
                                  LD, counts + 2, lo, nn));
  else if (p->pi <= 4) HGP_TRY(fused_tiers<4>(c, F, L));
  else HGP_TRY(fused_tiers<16>(c, F, L));
  uint32_t hc[8];
  HGP_TRY(read_back(c, counts, sizeof(hc), hc));
  if (hc[3]) {   // second pool, exactly the recorded counts of the pool-overflow nodes
    HGP_TRY(launch(c, "list_cnt_sum", k_list_cnt_sum, dim3(c->sm_count), dim3(256), 0, (const uint32_t *)LP,
                   (const uint32_t *)(counts + 3), (const uint32_t *)cnt, lo, misc + 3));
    uint64_t need = 0;
    HGP_TRY(read_u64(c, (const uint64_t *)(misc + 3), &need));
    uint32_t *pool2 = scratch_raw<uint32_t>(c, need ? need : 1, &st);
    if (st) return st;
    FusedJob F2 = F;
    F2.pool = pool2; F2.pool_cap = need ? need : 1; F2.pool_cursor = misc + 2;
    F2.start_bias = (uint64_t)(pool2 - pool);
    F2.pool_list = LA; F2.pool_count = counts + 6;
    TierLists L2{LP, counts + 3, hc[3], LA, counts + 4, LM, counts + 5, LD, counts + 2, false};
    if (p->pi <= 4) HGP_TRY(fused_tiers<4>(c, F2, L2));
    else HGP_TRY(fused_tiers<16>(c, F2, L2));
    HGP_TRY(read_back(c, counts, sizeof(hc), hc));
    if (hc[6]) return set_error(HGP_E_INTERNAL, "fused a2+a3: exact second pool overflowed");
  }
  if (hc[2] && !all_unfused && !c->opt.no_hub) {   // hubs: key-partitioned shared tables (hub.cu); what they leave -> LA
    HGP_TRY(hub_tier(c, F, LD, counts + 2, hc[2], LA, counts + 8));
    HGP_TRY(read_back(c, counts + 8, 4, &hc[2]));
    LD = LA;
    HGP_CUDA(cudaMemcpyAsync(counts + 2, counts + 8, 4, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (hc[2]) {   // unfused a2 + a3 for the nodes no fused tier could take (same results)
    uint32_t md = 0;
    HGP_TRY(nbrs_for_list(c, g, lo, LD, counts + 2, hc[2], pool, start, cnt, &md));
    ScoreJob J3 = J;
    J3.nb_off = nullptr; J3.nb_start = start; J3.nb_len = cnt; J3.nbr = pool;
    HGP_TRY(score_list_segments(c, J3, hc[2], md, LD, counts + 2));
  }
  HGP_TRY(score_finish(c));
  if (!out) {   // leave N(n) in the pool: segment n = pool[start[n] .. + cnt[n]) (relative to lo)
    HGP_CUDA(cudaMemsetAsync(misc + 3, 0, 8, c->stream));
    HGP_TRY(launch(c, "cnt_sum", k_cnt_sum, dim3(c->sm_count), dim3(256), 0, (const uint32_t *)cnt, nn, misc + 3));
    uint64_t V = 0;
    HGP_TRY(read_u64(c, (const uint64_t *)(misc + 3), &V));
    view->start = start; view->len = cnt; view->nbr = pool; view->V = V;
    return HGP_OK;
  }
  out->lo = lo;
  out->hi = hi;
  out->off = dalloc_n<uint64_t>(c, (size_t)nn + 1, &st);
  if (st) return st;
  uint64_t V = 0;
  HGP_TRY(scan_exclusive(c, InU32{cnt}, nn, out->off, &V));
  out->V = V;
  out->nbr = dalloc_n<uint32_t>(c, V, &st);
  if (st) return st;
  unsigned int *d_max = counts + 7;
  HGP_TRY(launch(c, "fused_pack", k_seg_pack_flat, dim3(8u * c->sm_count), dim3(256), 0, (const uint32_t *)pool,
                 (const uint64_t *)start, (const uint32_t *)cnt, (const uint64_t *)out->off, nn, V, out->nbr, d_max));
  uint32_t mx = 0;
  HGP_TRY(read_back(c, d_max, 4, &mx));
  out->max_deg = mx;
  return HGP_OK;
}


}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_neighbors_and_scores(hgp_ctx *c, const hgp_csr *g, const hgp_params *p, uint32_t lo,
                                               uint32_t hi, hgp_nbrs *nb, hgp_cand *cand) {
  if (!c || !g || !p || !nb || !cand) return set_error(HGP_E_ARG, "hgp_neighbors_and_scores: null argument");
  if (lo > hi || hi > g->N) return set_error(HGP_E_ARG, "hgp_neighbors_and_scores: bad node range");
  ApiScope scope(c);
  hgp_status s = hi > lo ? nbrs_score_fused(c, g, p, lo, hi, nb, cand, nullptr) : HGP_E_INTERNAL;
  if (s == HGP_OK) return HGP_OK;
  if (s != HGP_E_INTERNAL) { free_nbrs(c, nb); return s; }
  // unfused path: a2 then a3 (identical results)
  free_nbrs(c, nb);
  HGP_TRY(hgp_unique_neighbors(c, g, lo, hi, nb));
  s = score_run(c, g, nb, p, cand, nullptr, nullptr);
  if (s != HGP_OK) free_nbrs(c, nb);
  return s;
}

__global__ void k_node_work(const uint64_t *inc_off, const uint32_t *inc, const uint64_t *edge_off, uint32_t N,
                            uint64_t *work) {
  const uint32_t lane = lane_id();
  for (uint32_t n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += gridDim.x * (blockDim.x >> 5)) {
    uint64_t s = 0;
    for (uint64_t k = inc_off[n] + lane; k < inc_off[n + 1]; k += 32) {
      const uint32_t e = inc[k];
      s += edge_off[e + 1] - edge_off[e];
    }
    s = warp_sum(s);
    if (lane == 0) work[n] = s + 1;                              // +1: every node costs something
  }
}

__global__ void k_split(const uint64_t *prefix, uint32_t N, uint32_t world, uint32_t *bounds) {
  const uint32_t r = threadIdx.x;
  if (r > world) return;
  if (r == 0) { bounds[0] = 0; return; }
  if (r == world) { bounds[world] = N; return; }
  const uint64_t target = (prefix[N] * r + world - 1) / world;
  uint32_t a = 0, b = N;                                          // first n with prefix[n] >= target
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (prefix[mid] < target) a = mid + 1; else b = mid;
  }
  bounds[r] = a;
}

extern "C" hgp_status hgp_shard_bounds(hgp_ctx *c, const hgp_csr *g, uint32_t world, uint32_t *bounds) {
  if (!c || !g || !bounds || world == 0 || world > 1024) return set_error(HGP_E_ARG, "hgp_shard_bounds: bad argument");
  ApiScope scope(c);
  hgp_status st = HGP_OK;
  const uint32_t N = g->N;
  uint64_t *work = scratch_raw<uint64_t>(c, N ? N : 1, &st);
  uint64_t *prefix = scratch_raw<uint64_t>(c, (size_t)N + 1, &st);
  uint32_t *db = scratch_raw<uint32_t>(c, world + 1, &st);
  if (st) return st;
  const uint32_t grid = N ? (div_up(N, 8) < 16u * c->sm_count ? div_up(N, 8) : 16u * c->sm_count) : 0;
  HGP_TRY(launch(c, "node_work", k_node_work, dim3(grid), dim3(256), 0, (const uint64_t *)g->inc_off,
                 (const uint32_t *)g->inc, (const uint64_t *)g->edge_off, N, work));
  HGP_TRY(scan_exclusive(c, InU64{work}, N, prefix, nullptr));
  HGP_TRY(launch(c, "split", k_split, dim3(1), dim3(world + 1), 0, (const uint64_t *)prefix, N, world, db));
  return read_back(c, db, 4 * ((size_t)world + 1), bounds);
}

extern "C" hgp_status hgp_coarsen_level0(hgp_ctx *c, const hgp_csr *g, const hgp_params *p, hgp_cand *cand,
                                         uint32_t *match, uint32_t *gamma, hgp_nbrs *nb, hgp_csr *coarse,
                                         hgp_nbrs *coarse_nb, hgp_level_stats *stats) {
  if (!c || !g || !p || !match || !gamma || !coarse || !coarse_nb)
    return set_error(HGP_E_ARG, "hgp_coarsen_level0: null argument");
  if (p->pi < 1 || p->pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "pi must be in [1,16]");
  ApiScope scope(c);
  hgp_status st = HGP_OK;
  if (!cand) {
    cand = scratch_raw<hgp_cand>(c, (size_t)g->N * p->pi, &st);
    if (st) return st;
  }
  uint32_t *per = scratch_zero<uint32_t>(c, HGP_MAX_PI, &st);
  if (st) return st;
  // nb == NULL: the level's N(n) stays in the fused kernel's pool and a5 reads it there (no
  // compaction pass); otherwise it is returned as a CSR with the flags a3 set.
  hgp_nbrs local{};
  hgp_nbrs *use = nb ? nb : &local;
  SegView view{};
  bool have_view = false;
  HGP_CUDA(cudaEventRecord(c->ev[0], c->stream));
  if (!nb && g->N) {
    hgp_status s = nbrs_score_fused(c, g, p, 0, g->N, nullptr, cand, &view);
    if (s == HGP_OK) have_view = true;
    else if (s != HGP_E_INTERNAL) return s;
  }
  if (!have_view) HGP_TRY(hgp_neighbors_and_scores(c, g, p, 0, g->N, use, cand));
  HGP_CUDA(cudaEventRecord(c->ev[1], c->stream));
  auto cleanup = [&]() { if (!have_view && !nb) free_nbrs(c, &local); };
  hgp_status s = hgp_match(c, cand, g->N, p->pi, match, per);
  if (s == HGP_OK && (p->flags & HGP_FLAG_LEFTOVER))
    s = leftover_impl(c, cand, g->N, p->pi, g->node_w, g->in_mu, p->omega, p->delta, match, nullptr);
  if (s != HGP_OK) { cleanup(); if (nb) free_nbrs(c, nb); return s; }
  HGP_CUDA(cudaEventRecord(c->ev[2], c->stream));
  s = contract_impl(c, g, have_view ? nullptr : use, match, gamma, coarse, coarse_nb, stats, have_view ? &view : nullptr);
  if (s != HGP_OK) { free_csr(c, coarse); free_nbrs(c, coarse_nb); cleanup(); if (nb) free_nbrs(c, nb); return s; }
  HGP_CUDA(cudaEventRecord(c->ev[3], c->stream));
  HGP_CUDA(cudaEventSynchronize(c->ev[3]));
  if (stats) {
    stats->N = g->N; stats->E = g->E; stats->P = g->P; stats->V = have_view ? view.V : use->V;
    uint32_t hper[HGP_MAX_PI];
    HGP_TRY(read_back(c, per, sizeof(hper), hper));
    for (int i = 0; i < HGP_MAX_PI; ++i) stats->matched_per_round[i] = i < (int)p->pi ? hper[i] : 0;
    cudaEventElapsedTime(&stats->ms[0], c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&stats->ms[1], c->ev[1], c->ev[2]);
    cudaEventElapsedTime(&stats->ms[2], c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&stats->ms[3], c->ev[0], c->ev[3]);
  }
  cleanup();
  return HGP_OK;
}
