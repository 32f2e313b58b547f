// contract.cu — a5: coarse hypergraph construction (§5.5; §3).
//
//  gamma   rep(n) <=> match(n) = NONE or n < match(n); coarse id = exclusive scan of rep
//          (ascending min member); gamma(n) = cid(min(n, match(n))); size' = sum of sizes.
//  edges   per fine edge (in its own oversized slot): map pins by gamma, sort the
//          src and dst blocks, D' = unique dst, S' = unique src \ D' (duplicates kept in dst,
//          P:831); dropped iff D' empty and |S'| <= 1 (reading #14).
//  merge   parallel edges (identical (S',D')) are found through a global hash table keyed by a
//          64-bit fingerprint and verified element by element; the class representative is the
//          minimum fine edge id (atomicMin), omega' = sum omega, mu' = sum mu (reading #12);
//          coarse edges are ordered by representative.
//  incid.  rebuilt by the a1 transpose (canonical in-first lists, in_mu' = sum mu').
//  N'      per coarse node: gamma(N(a) ∪ N(b)) in a hash set with an OR-ed purge flag per key;
//          flagged keys and the node itself are dropped (reading #7).
#include "csr_impl.cuh"
#include "hashset.cuh"
#include "lbs.cuh"
#include "scan.cuh"
#include "sort.cuh"

namespace hgp {

constexpr int kErrMatch = 10;

__global__ void k_rep(const uint32_t *match, uint32_t N, uint32_t *rep, uint64_t *err) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const uint32_t m = match[n];
    if (m != kNone && (m >= N || m == n || match[m] != n)) report_min(err, kErrMatch, n);
    rep[n] = (m == kNone || n < m) ? 1u : 0u;
  }
}

__global__ void k_gamma(const uint32_t *match, const uint64_t *cid, const uint32_t *node_w, uint32_t N,
                        uint32_t *gamma, uint32_t *cw, uint32_t *mem0, uint32_t *mem1) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const uint32_t m = match[n];
    const uint32_t lo = (m == kNone || n < m) ? n : m;
    const uint32_t c = (uint32_t)cid[lo];
    gamma[n] = c;
    if (cw) atomicAdd(&cw[c], node_w[n]);
    if (lo == n) { mem0[c] = n; mem1[c] = m; }
  }
}

__global__ void __launch_bounds__(kLbsThreads) k_map_pins(const uint32_t *pins, const uint32_t *gamma, uint64_t P,
                                                          uint32_t *out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (uint64_t)gridDim.x * blockDim.x)
    out[p] = gamma[pins[p]];
}

struct EdgeSeg2 {   // segment 2e = src(e), 2e+1 = dst(e) of the fine layout
  const uint64_t *off;
  const uint32_t *nsrc;
  __device__ void operator()(uint64_t i, uint64_t &beg, uint32_t &len) const {
    const uint64_t e = i >> 1;
    const uint64_t lo = off[e], hi = off[e + 1], s = lo + nsrc[e];
    if (i & 1) { beg = s; len = (uint32_t)(hi - s); }
    else { beg = lo; len = (uint32_t)(s - lo); }
  }
};

__device__ __forceinline__ uint64_t fp_mix(uint64_t h, uint32_t x, uint32_t i) {
  return h + splitmix64(((uint64_t)x << 32) ^ (uint64_t)i * 0xD6E8FEB86659FD93ull);
}

// Unique + src\dst filtering in place; layout [S'][D'] from off[e]; warp per edge.
__global__ void k_edge_unique(const uint64_t *off, const uint32_t *nsrc, uint32_t E, uint32_t *x, uint32_t *cnsrc,
                              uint32_t *csize, uint8_t *keep, uint64_t *fp) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t e = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < E; e += nw) {
    const uint64_t lo = off[e], hi = off[e + 1], s = lo + nsrc[e];
    // S' = unique src not present in the (sorted) dst block
    uint32_t ns = 0;
    uint32_t prev = kNone;   // last element of the previous chunk
    for (uint64_t base = lo; base < s; base += 32) {
      const uint64_t j = base + lane;
      uint32_t v = j < s ? x[j] : kNone;
      const uint32_t before = __shfl_up_sync(0xFFFFFFFFu, v, 1);
      const uint32_t left = lane == 0 ? prev : before;
      bool k = j < s && v != left;
      if (k) {
        uint64_t a = s, b = hi;
        while (a < b) {
          const uint64_t m = (a + b) >> 1;
          if (x[m] < v) a = m + 1; else b = m;
        }
        if (a < hi && x[a] == v) k = false;
      }
      prev = __shfl_sync(0xFFFFFFFFu, v, 31);
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, k);
      __syncwarp();
      if (k) x[lo + ns + __popc(bal & lt)] = v;
      ns += __popc(bal);
      __syncwarp();
    }
    // D' = unique dst, moved to lo + ns (never overtakes the read position: ns <= s - lo)
    uint32_t nd = 0;
    prev = kNone;
    for (uint64_t base = s; base < hi; base += 32) {
      const uint64_t j = base + lane;
      const uint32_t v = j < hi ? x[j] : kNone;
      const uint32_t before = __shfl_up_sync(0xFFFFFFFFu, v, 1);
      const uint32_t left = lane == 0 ? prev : before;
      const bool k = j < hi && v != left;
      prev = __shfl_sync(0xFFFFFFFFu, v, 31);
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, k);
      __syncwarp();
      if (k) x[lo + ns + nd + __popc(bal & lt)] = v;
      nd += __popc(bal);
      __syncwarp();
    }
    const bool kp = !(nd == 0 && ns <= 1);
    // fingerprint of (|S'|, S', D')
    uint64_t h = 0;
    if (kp)
      for (uint32_t i = lane; i < ns + nd; i += 32) h = fp_mix(h, x[lo + i], i);
    h = warp_sum(h);
    if (lane == 0) {
      cnsrc[e] = ns;
      csize[e] = ns + nd;
      keep[e] = kp;
      fp[e] = splitmix64(h ^ ((uint64_t)ns << 40) ^ (uint64_t)(ns + nd));
    }
  }
}

// Entries k of the merge: the fine edge eid[k] (identity when eid == nullptr) whose coarse pins
// are x[off[k] .. off[k] + csize[k]); keep == nullptr: every entry is kept. Entries ascend by
// fine edge id, so the class representative (the minimum fine id) is the minimum entry.
struct MergeJob {
  const uint64_t *off;
  const uint32_t *x, *cnsrc, *csize;
  const uint8_t *keep;
  const uint64_t *fp;
  const uint32_t *eid;
  uint32_t E;                // entries
  uint32_t *owner;     // table slots: edge id of the first inserter (kEmpty = free)
  uint32_t *minrep;    // per slot: min edge id of the class
  uint32_t *slot_of;   // per edge
  uint32_t log2t;
};

__device__ __forceinline__ bool same_edge(const MergeJob &M, uint32_t a, uint32_t b) {
  if (M.fp[a] != M.fp[b] || M.cnsrc[a] != M.cnsrc[b] || M.csize[a] != M.csize[b]) return false;
  const uint32_t *pa = M.x + M.off[a], *pb = M.x + M.off[b];
  for (uint32_t i = 0; i < M.csize[a]; ++i)
    if (pa[i] != pb[i]) return false;
  return true;
}

__global__ void k_merge_insert(MergeJob M) {
  const uint32_t mask = (1u << M.log2t) - 1;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < M.E; e += gridDim.x * blockDim.x) {
    if (M.keep && !M.keep[e]) continue;
    uint32_t slot = (uint32_t)(M.fp[e] >> 7) & mask;
    while (true) {
      uint32_t o = *(volatile uint32_t *)&M.owner[slot];
      if (o == kEmpty) {
        o = atomicCAS(&M.owner[slot], kEmpty, e);
        if (o == kEmpty) break;
      }
      if (same_edge(M, o, e)) break;
      slot = (slot + 1) & mask;
    }
    M.slot_of[e] = slot;
    atomicMin(&M.minrep[slot], e);
  }
}

__global__ void k_merge_resolve(MergeJob M, uint32_t *rep, uint32_t *is_rep) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < M.E; e += gridDim.x * blockDim.x) {
    const uint32_t r = (!M.keep || M.keep[e]) ? M.minrep[M.slot_of[e]] : kNone;
    rep[e] = r;
    is_rep[e] = r == e;
  }
}

__global__ void k_coarse_edge_attrs(const uint32_t *rep, const uint64_t *ceid, const uint32_t *edge_w,
                                    const uint32_t *edge_mu, const uint32_t *cnsrc, const uint32_t *csize, uint32_t E,
                                    const uint32_t *eid, uint32_t *cw, uint32_t *cmu, uint32_t *c_nsrc,
                                    uint32_t *c_size) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint32_t r = rep[e];
    if (r == kNone) continue;
    const uint32_t ce = (uint32_t)ceid[r];
    const uint32_t fe = eid ? eid[e] : e;                          // the fine edge of entry e
    atomicAdd(&cw[ce], edge_w[fe]);
    atomicAdd(&cmu[ce], edge_mu[fe]);
    if (r == e) { c_nsrc[ce] = cnsrc[e]; c_size[ce] = csize[e]; }
  }
}

__global__ void k_coarse_edge_pack(const uint32_t *rep, const uint64_t *ceid, const uint64_t *off, const uint32_t *x,
                                   const uint32_t *csize, const uint64_t *coff, uint32_t E, uint32_t *cpins,
                                   unsigned int *maxe) {
  const uint32_t lane = lane_id();
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  uint32_t mx = 0;
  for (uint64_t e = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < E; e += nw) {
    if (rep[e] != e) continue;
    const uint32_t n = csize[e];
    const uint32_t *src = x + off[e];
    uint32_t *dst = cpins + coff[ceid[e]];
    for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
    mx = max(mx, n);
  }
  mx = warp_max(mx);
  if (lane == 0) atomicMax(maxe, mx);
}

// ---------------------------------------------------------------- coarse neighbours
struct CNbrJob {
  const uint32_t *mem0, *mem1;
  const uint64_t *nb_off;      // CSR offsets, or nullptr when nb_start/nb_len describe the segments
  const uint64_t *nb_start;
  const uint32_t *nb_len;
  const uint32_t *nbr;
  const uint32_t *gamma;
  const uint64_t *bound_off;   // exclusive scan of |N(a)|+|N(b)| (oversized slots)
  uint32_t *pool;              // [V]
  uint32_t *cnt;               // [Nc]
  const uint32_t *list;        // coarse nodes for this tier (nullptr: all, filtered by cap)
  const uint32_t *list_count;
  uint32_t Nc;
  uint32_t cap;                // tier capacity (entries)
  uint32_t log2s;
  uint32_t *gtab;              // global tables (keys | flags) when not in smem
  unsigned long long *purged;
  unsigned long long *tiers;   // work counters (hgp_tier_counts)
  int tier;
  uint32_t cbase;              // coarse id of local coarse node 0 (a range of coarse nodes)
  uint32_t *nbr_w;             // in place (pool == nullptr): N'(c) overwrites N(a)'s then N(b)'s
};                             // segment, which only c's CTA reads (each fine node has one c)

// Where entry pos of N'(c) goes: the oversized pool slot, or in place over N(a) ‖ N(b).
__device__ __forceinline__ uint32_t *cnbr_out(const CNbrJob &J, uint64_t base, uint64_t a0, uint64_t na, uint64_t b0,
                                              uint64_t pos) {
  if (J.pool) return J.pool + base + pos;
  return J.nbr_w + (pos < na ? a0 + pos : b0 + (pos - na));
}

// insert key with an OR-ed flag kept in bit 31 of the slot (ids < 2^31 - 1, kEmpty masks to
// 0x7FFFFFFF which is never an id); returns true if this call inserted the key.
__device__ __forceinline__ bool hs_insert_flagged(uint32_t *keys, uint32_t log2s, uint32_t key, bool flag,
                                                  uint32_t *slot_out) {
  const uint32_t mask = (1u << log2s) - 1;
  uint32_t s = hash_slot(key, log2s);
  volatile uint32_t *vk = keys;
  while (true) {
    uint32_t k = vk[s];
    if (k == kEmpty) {
      k = atomicCAS(&keys[s], kEmpty, flag ? (key | kPurge) : key);
      if (k == kEmpty) { *slot_out = s; return true; }
    }
    if ((k & kIdMask) == key) {
      if (flag && !(k & kPurge)) atomicOr(&keys[s], kPurge);
      *slot_out = s;
      return false;
    }
    s = (s + 1) & mask;
  }
}

// One CTA per coarse node c = {a, b}: gamma(N(a) ∪ N(b)) into a hash set whose slots carry an
// OR-ed purge flag in bit 31; then the unflagged keys other than c are compacted (two ballot
// passes over the table, warp-owned ranges, no atomics) into c's oversized pool slot.
template <int THREADS, bool SMEM>
__global__ void __launch_bounds__(THREADS) k_coarse_nbrs(CNbrJob J) {
  extern __shared__ uint32_t dyn[];
  constexpr uint32_t NW = THREADS / 32;
  __shared__ uint32_t s_wcnt[NW];
  __shared__ uint32_t s_n, s_out;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t log2s = J.log2s, S = 1u << log2s;
  uint32_t *keys = SMEM ? dyn : J.gtab + ((size_t)blockIdx.x << log2s);
  uint16_t *slist = reinterpret_cast<uint16_t *>(dyn + S);          // SMEM: slots inserted (<= S/2)
  const uint32_t keys_s = SMEM ? opaque_u32(smem_u32addr(keys)) : 0u;
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t total = J.list_count ? *J.list_count : J.Nc;
  uint64_t purged = 0;
  uint32_t done = 0;
  if (SMEM) {   // cleared once; afterwards every node leaves exactly the slots it used to clear
    for (uint32_t i = tid; i < S / 4; i += THREADS)
      reinterpret_cast<uint4 *>(keys)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    if (tid == 0) { s_n = 0; s_out = 0; }
    __syncthreads();
  }
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const uint32_t c = J.list ? J.list[t] : t;
    const uint32_t a = J.mem0[c], b = J.mem1[c];
    uint64_t a0, a1, b0 = 0, b1 = 0;
    if (J.nb_off) {
      a0 = J.nb_off[a]; a1 = J.nb_off[a + 1];
      if (b != kNone) { b0 = J.nb_off[b]; b1 = J.nb_off[b + 1]; }
    } else {
      a0 = J.nb_start[a]; a1 = a0 + J.nb_len[a];
      if (b != kNone) { b0 = J.nb_start[b]; b1 = b0 + J.nb_len[b]; }
    }
    const uint64_t na = a1 - a0, nbn = b1 - b0;
    if (!J.list && na + nbn > J.cap) continue;                      // larger tier (uniform)
    // global tables: only nextpow2(2 (|N(a)| + |N(b)| + 1)) slots of the CTA's region
    uint32_t nlog = log2s;
    if (!SMEM) {
      nlog = 6;
      while ((1ull << nlog) < 2 * (na + nbn + 1) && nlog < log2s) ++nlog;
    }
    const uint32_t Sn = 1u << nlog, nmask = Sn - 1;
    if (!SMEM) {
      for (uint32_t i = tid; i < Sn / 4; i += THREADS)
        reinterpret_cast<uint4 *>(keys)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncthreads();
    }
    // 4 entries per thread in flight: nbr loads, then the gamma gathers, then the inserts
    for (uint64_t kb = 0; kb < na + nbn; kb += 4 * THREADS) {       // CTA-uniform trip count
      const uint64_t k0 = kb + tid;
      uint32_t v[4], gm[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t k = k0 + (uint64_t)u * THREADS;
        v[u] = k < na + nbn ? (k < na ? J.nbr[a0 + k] : J.nbr[b0 + (k - na)]) : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) gm[u] = v[u] != kEmpty ? __ldg(J.gamma + (v[u] & kIdMask)) : kEmpty;
      uint32_t nslot[4], newm = 0;                                  // new keys: slots, mask (SMEM)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (v[u] == kEmpty) continue;
        const bool fl = (v[u] & kPurge) != 0;
        purged += fl;
        if constexpr (SMEM) {
          uint32_t slot = hash_slot(gm[u], nlog);
          uint32_t k = lds_hint_u32(keys_s + 4 * slot);
          while (true) {
            if (k == kEmpty) {
              k = cas_u32(keys_s + 4 * slot, kEmpty, fl ? (gm[u] | kPurge) : gm[u]);
              if (k == kEmpty) { nslot[u] = slot; newm |= 1u << u; break; }   // a new key
            }
            if ((k & kIdMask) == gm[u]) {
              if (fl && !(k & kPurge)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(keys_s + 4 * slot), "r"(kPurge) : "memory");
              break;
            }
            slot = (slot + 1) & nmask;
            k = lds_hint_u32(keys_s + 4 * slot);
          }
        } else {
          uint32_t slot;
          hs_insert_flagged(keys, nlog, gm[u], fl, &slot);
        }
      }
      if constexpr (SMEM) {   // the new keys' slots to the list: one shared atomic per warp
        const uint32_t nnew = __popc(newm);
        const uint32_t incl = warp_incl_scan(nnew);
        uint32_t base = 0;
        if (lane == 31 && incl) base = atomicAdd(&s_n, incl);
        base = __shfl_sync(0xFFFFFFFFu, base, 31) + incl - nnew;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((newm >> u) & 1u) slist[base + __popc(newm & ((1u << u) - 1))] = (uint16_t)nslot[u];
      }
    }
    __syncthreads();
    const uint64_t base = J.pool ? J.bound_off[c] : 0;
    if constexpr (SMEM) {
      // the inserted slots: unflagged keys other than c go to the pool (warp chunks claim their
      // output positions with one shared atomic; the segment is a set), every slot is cleared
      const uint32_t nl = s_n;
      for (uint32_t i0 = w * 32; i0 < nl; i0 += THREADS) {
        const uint32_t i = i0 + lane;
        const bool valid = i < nl;
        const uint32_t slot = valid ? slist[i] : 0u;
        const uint32_t k = valid ? keys[slot] : kEmpty;
        const bool keep = valid && !(k & kPurge) && k != c + J.cbase;   // kEmpty has bit 31 set
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
        uint32_t wpos = 0;
        if (lane == 0 && bal) wpos = atomicAdd(&s_out, (uint32_t)__popc(bal));
        wpos = __shfl_sync(0xFFFFFFFFu, wpos, 0);
        if (keep) *cnbr_out(J, base, a0, na, b0, wpos + __popc(bal & lt)) = k;
        if (valid) keys[slot] = kEmpty;
      }
      __syncthreads();
      if (tid == 0) { J.cnt[c] = s_out; ++done; s_n = 0; s_out = 0; }
      __syncthreads();
    } else {
      // global tables: unflagged keys != c by two ballot sweeps over the table
      const uint32_t per_w = Sn / NW, w0 = w * per_w;
      uint32_t mine = 0;
      for (uint32_t sb = w0; sb < w0 + per_w; sb += 32) {
        const uint32_t k = keys[sb + lane];
        mine += __popc(__ballot_sync(0xFFFFFFFFu, !(k & kPurge) && k != c + J.cbase));   // kEmpty has bit 31 set
      }
      if (lane == 0) s_wcnt[w] = mine;
      __syncthreads();
      uint32_t wpos = 0, tot = 0;
      for (uint32_t q = 0; q < NW; ++q) { const uint32_t x = s_wcnt[q]; if (q < w) wpos += x; tot += x; }
      for (uint32_t sb = w0; sb < w0 + per_w; sb += 32) {
        const uint32_t k = keys[sb + lane];
        const bool keep = !(k & kPurge) && k != c + J.cbase;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
        if (keep) *cnbr_out(J, base, a0, na, b0, wpos + __popc(bal & lt)) = k;
        wpos += __popc(bal);
      }
      if (tid == 0) { J.cnt[c] = tot; ++done; }
      __syncthreads();
    }
  }
  if (tid == 0) tier_add(J.tiers, J.tier, done);
  purged = warp_sum(purged);
  if ((tid & 31) == 0 && purged) atomicAdd(J.purged, (unsigned long long)purged);
}

struct BoundIn {   // |N(a)| + |N(b)| per coarse node
  const uint32_t *mem0, *mem1;
  const uint64_t *nb_off;
  const uint32_t *nb_len;
  __device__ uint64_t len(uint32_t n) const { return nb_off ? nb_off[n + 1] - nb_off[n] : nb_len[n]; }
  __device__ uint64_t operator()(uint64_t c) const {
    const uint32_t a = mem0[c], b = mem1[c];
    return len(a) + (b == kNone ? 0 : len(b));
  }
};

__global__ void k_cnbr_classify(const uint64_t *bound_off, uint32_t Nc, uint32_t capA, uint32_t capA2, uint32_t capM,
                                uint32_t capB, uint32_t *listA2, uint32_t *listM, uint32_t *listB, uint32_t *listC,
                                uint32_t *counts, unsigned long long *maxb) {
  uint64_t mx = 0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < Nc; c += gridDim.x * blockDim.x) {
    const uint64_t d = bound_off[c + 1] - bound_off[c];
    if (d > capA) {
      if (d <= capA2) listA2[atomicAdd(&counts[3], 1u)] = c;
      else if (d <= capM) listM[atomicAdd(&counts[0], 1u)] = c;
      else if (d <= capB) listB[atomicAdd(&counts[1], 1u)] = c;
      else { listC[atomicAdd(&counts[2], 1u)] = c; mx = d > mx ? d : mx; }
    }
  }
  mx = warp_max(mx);
  if (lane_id() == 0 && mx) atomicMax(maxb, (unsigned long long)mx);
}

__global__ void k_list_max_bound(const uint64_t *bound_off, const uint32_t *list, const uint32_t *count,
                                 unsigned long long *maxb) {
  uint64_t mx = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < *count; i += gridDim.x * blockDim.x) {
    const uint32_t c = list[i];
    mx = max(mx, bound_off[c + 1] - bound_off[c]);
  }
  mx = warp_max(mx);
  if (lane_id() == 0 && mx) atomicMax(maxb, (unsigned long long)mx);
}

// The pack as a flat copy balanced by entries, not by node: warp w copies the output positions
// [Vc w / W, Vc (w+1) / W), walking the coarse nodes they span (one binary search over off for the
// first). A warp per node left the hubs' ~10^6-entry neighbourhoods to single warps (C4: 9.4 ms for
// ~10 GB). INPLACE: N'(c) is the first cnt[c] entries of N(a)'s segment followed by N(b)'s;
// else the oversized pool slot at bound_off[c].
template <bool INPLACE>
__global__ void k_cnbr_pack_flat(CNbrJob J, const uint32_t *pool, const uint64_t *bound_off, const uint64_t *off,
                                 uint32_t Nc, uint64_t Vc, uint32_t *nbr, unsigned int *maxdeg) {
  const uint32_t lane = lane_id();
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t mx = 0;                                                  // max |N'(c)|: grid-stride over c
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < Nc; c += gridDim.x * blockDim.x) mx = max(mx, J.cnt[c]);
  mx = warp_max(mx);
  if (lane == 0 && mx) atomicMax(maxdeg, mx);
  const uint64_t lo = Vc * wid / W, hi = Vc * (wid + 1) / W;
  if (lo >= hi) return;
  uint32_t a = 0, b = Nc;                                           // last c with off[c] <= lo
  while (b - a > 1) {
    const uint32_t m = (a + b) >> 1;
    if (off[m] <= lo) a = m; else b = m;
  }
  uint64_t pos = lo;
  for (uint32_t c = a; pos < hi; ++c) {
    const uint64_t s0 = off[c], s1 = off[c + 1];
    if (s1 <= pos) continue;                                        // (empty nodes)
    const uint32_t i0 = (uint32_t)(pos - s0), i1 = (uint32_t)((s1 < hi ? s1 : hi) - s0);
    uint64_t a0 = 0, na = 0, b0 = 0;
    const uint32_t *src = nullptr;
    if (INPLACE) {
      const uint32_t ma = J.mem0[c], mb = J.mem1[c];
      a0 = J.nb_start[ma];
      na = J.nb_len[ma];
      b0 = mb == kNone ? 0 : J.nb_start[mb];
    } else {
      src = pool + bound_off[c];
    }
    uint32_t *dst = nbr + s0;
    for (uint32_t j0 = i0; j0 < i1; j0 += 128) {                    // 4 loads in flight per lane
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = j0 + u * 32 + lane;
        v[u] = i < i1 ? (INPLACE ? J.nbr_w[i < na ? a0 + i : b0 + (i - na)] : src[i]) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { const uint32_t i = j0 + u * 32 + lane; if (i < i1) dst[i] = v[u]; }
    }
    pos = s0 + i1;
  }
}

__global__ void k_count_kept(const uint32_t *rep, uint32_t E, uint32_t *out) {
  uint32_t s = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) s += rep[e] != kNone;
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(out, s);
}

// ---- hub coarse nodes (|N(a)| + |N(b)| above tier B), key-partitioned like the fused hub tier
// (hub.cu): the entries gamma(v) | flag are bucketed by a hash of gamma(v) into k(c) partitions
// whose entry counts all fit half of an 8192-slot table (the size pass doubles k until they do,
// so an item can never overflow: no fallback after N'(c) is partly written in place); one CTA
// per partition deduplicates its bucket with OR-ed purge flags and appends its unflagged keys to
// N'(c) (one atomic per partition on c's counter). Same set as tiers A-C (a union of per-key
// decisions that do not depend on the partition).
constexpr uint32_t kCHLog = 13, kCHCap = 1u << (kCHLog - 1), kCHMaxParts = 4096, kCHThreads = 256;

__device__ __forceinline__ uint32_t chub_part(uint32_t m, uint32_t k) {   // independent of hash_slot
  uint32_t h = m * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0xC2B2AE3Du;
  h ^= h >> 13;
  return __umulhi(h, k);
}

struct CHubJob {
  CNbrJob J;
  const uint32_t *list, *list_count;   // coarse nodes (relative ids)
  uint32_t *hk;                        // [list] partitions (0: left to tier C)
  uint64_t *hb;                        // [list] entries |N(a)| + |N(b)|
  const uint64_t *item_off, *vis_off;  // [list] exclusive scans of hk / hb
  uint32_t *ibase, *ilen, *inode;      // [items] bucket (relative to vis_off), length, list index
  uint32_t *bkey;                      // [sum hb] gamma(v) | purge flag of v
  uint32_t *hcnt;                      // [list] |N'(c)| so far
  uint32_t *lu, *lu_count;             // -> tier C
};

// entries of c = {a, b}: N(a) then N(b)
struct CEntries {
  uint64_t a0, na, b0, n;
  __device__ CEntries(const CNbrJob &J, uint32_t c) {
    const uint32_t a = J.mem0[c], b = J.mem1[c];
    uint64_t a1, b1 = 0;
    b0 = 0;
    if (J.nb_off) { a0 = J.nb_off[a]; a1 = J.nb_off[a + 1]; if (b != kNone) { b0 = J.nb_off[b]; b1 = J.nb_off[b + 1]; } }
    else { a0 = J.nb_start[a]; a1 = a0 + J.nb_len[a]; if (b != kNone) { b0 = J.nb_start[b]; b1 = b0 + J.nb_len[b]; } }
    na = a1 - a0;
    n = na + (b1 - b0);
  }
  __device__ uint64_t at(uint64_t j) const { return j < na ? a0 + j : b0 + (j - na); }
};

// size (MODE 0): k(c) with every partition's entry count <= kCHCap; scatter (MODE 1): bucket
// offsets, then the entries into their buckets. One CTA per listed coarse node.
template <int MODE>
__global__ void __launch_bounds__(kCHThreads) k_chub_visit(CHubJob H) {
  constexpr uint32_t NW = kCHThreads / 32;
  __shared__ uint32_t s_h[kCHMaxParts];
  __shared__ uint32_t s_w[NW];
  __shared__ uint32_t s_max;
  const CNbrJob &J = H.J;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t total = *H.list_count;
  uint64_t purged = 0;
  for (uint32_t i = blockIdx.x; i < total; i += gridDim.x) {
    const uint32_t c = H.list[i];
    const CEntries X(J, c);
    const uint32_t self = c + J.cbase;
    uint32_t k = MODE == 0 ? (uint32_t)max((uint64_t)1, (X.n + kCHCap / 2 - 1) / (kCHCap / 2)) : H.hk[i];
    if (k == 0 || k > kCHMaxParts) {                                // CTA-uniform: tier C takes it
      if (MODE == 0 && tid == 0) { H.hk[i] = 0; H.hb[i] = 0; H.lu[atomicAdd(H.lu_count, 1u)] = c; }
      continue;
    }
    while (true) {
      for (uint32_t r = tid; r < k; r += kCHThreads) s_h[r] = 0;
      if (tid == 0) s_max = 0;
      __syncthreads();
      for (uint64_t j = tid; j < X.n; j += kCHThreads) {
        const uint32_t v = J.nbr[X.at(j)];
        if (MODE == 1) purged += (v & kPurge) != 0;                 // (hubs only: tier C counts its own)
        const uint32_t key = __ldg(J.gamma + (v & kIdMask));
        if (key != self) atomicAdd(&s_h[chub_part(key, k)], 1u);
      }
      __syncthreads();
      if (MODE == 1) break;
      uint32_t mx = 0;
      for (uint32_t r = tid; r < k; r += kCHThreads) mx = max(mx, s_h[r]);
      mx = __reduce_max_sync(0xFFFFFFFFu, mx);
      if (lane == 0) atomicMax(&s_max, mx);
      __syncthreads();
      const uint32_t m = s_max;
      __syncthreads();                                              // s_max / s_h rewritten next
      if (m <= kCHCap || 2 * k > kCHMaxParts) {
        if (tid == 0) {
          const bool fits = m <= kCHCap;
          H.hk[i] = fits ? k : 0;
          H.hb[i] = fits ? X.n : 0;
          H.hcnt[i] = 0;
          if (!fits) H.lu[atomicAdd(H.lu_count, 1u)] = c;
        }
        break;
      }
      k *= 2;
    }
    if (MODE == 1) {
      // bucket offsets: exclusive scan of the histogram; items; then the scatter with cursors
      const uint64_t it0 = H.item_off[i], vo = H.vis_off[i];
      const uint32_t per = (k + kCHThreads - 1) / kCHThreads, r0 = min(k, tid * per), r1 = min(k, r0 + per);
      uint32_t run = 0;
      for (uint32_t r = r0; r < r1; ++r) run += s_h[r];
      const uint32_t wincl = warp_incl_scan(run);
      if (lane == 31) s_w[w] = wincl;
      __syncthreads();
      uint32_t base = wincl - run;
#pragma unroll
      for (uint32_t q = 0; q < NW; ++q) base += q < w ? s_w[q] : 0u;
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t cn = s_h[r];
        H.ibase[it0 + r] = base;
        H.ilen[it0 + r] = cn;
        H.inode[it0 + r] = i;
        s_h[r] = base;                                              // own entries only: no race
        base += cn;
      }
      __syncthreads();
      for (uint64_t j = tid; j < X.n; j += kCHThreads) {
        const uint32_t v = J.nbr[X.at(j)];
        const uint32_t key = __ldg(J.gamma + (v & kIdMask));
        if (key == self) continue;
        const uint32_t pos = atomicAdd(&s_h[chub_part(key, k)], 1u);
        H.bkey[vo + pos] = key | (v & kPurge);
      }
      __syncthreads();                                              // s_h / s_w reused next node
    }
  }
  if (MODE == 1) {
    purged = warp_sum(purged);
    if (lane == 0 && purged) atomicAdd(J.purged, (unsigned long long)purged);
  }
}

// one CTA per partition: dedup with OR-ed flags, then the unflagged keys appended to N'(c)
__global__ void __launch_bounds__(kCHThreads) k_chub_items(CHubJob H, uint32_t nitems) {
  extern __shared__ __align__(16) uint32_t ckeys[];
  constexpr uint32_t NW = kCHThreads / 32, S = 1u << kCHLog, hmask = S - 1;
  __shared__ uint32_t s_w[NW];
  __shared__ uint32_t s_pos;
  const CNbrJob &J = H.J;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t keys_s = opaque_u32(smem_u32addr(ckeys));
  for (uint32_t j = tid; j < S / 4; j += kCHThreads) reinterpret_cast<uint4 *>(ckeys)[j] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
  __syncthreads();
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint32_t i = H.inode[it];
    const uint32_t c = H.list[i];
    const uint64_t bb = H.vis_off[i] + H.ibase[it];
    const uint32_t len = H.ilen[it];
    for (uint32_t j = tid; j < len; j += kCHThreads) {
      const uint32_t x = H.bkey[bb + j];
      const uint32_t key = x & kIdMask, fl = x & kPurge;
      uint32_t slot = hash_slot(key, kCHLog);
      uint32_t kk = lds_u32(keys_s + 4 * slot);
      while (true) {                                                // load <= 1/2: terminates
        if (kk == kEmpty) {
          kk = cas_u32(keys_s + 4 * slot, kEmpty, x);
          if (kk == kEmpty) break;
        }
        if ((kk & kIdMask) == key) {
          if (fl && !(kk & kPurge)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(keys_s + 4 * slot), "r"(kPurge) : "memory");
          break;
        }
        slot = (slot + 1) & hmask;
        kk = lds_u32(keys_s + 4 * slot);
      }
    }
    __syncthreads();
    // kept keys (unflagged; kEmpty has bit 31 set): count, one position claim, write + clear
    constexpr uint32_t SW = S / NW;                                 // warp w owns [w SW, (w+1) SW)
    uint32_t cnt = 0;
    for (uint32_t j = w * SW + lane; j < (w + 1) * SW; j += 32) cnt += !(ckeys[j] & kPurge);
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (lane == 0) s_w[w] = cnt;
    __syncthreads();
    if (tid == 0) {
      uint32_t t = 0;
      for (uint32_t q = 0; q < NW; ++q) t += s_w[q];
      s_pos = t ? atomicAdd(&H.hcnt[i], t) : 0u;
    }
    __syncthreads();
    const CEntries X(J, c);
    const uint64_t base = J.pool ? J.bound_off[c] : 0;
    uint32_t wpos = s_pos;
    for (uint32_t q = 0; q < w; ++q) wpos += s_w[q];
    const uint32_t lt = (1u << lane) - 1;
    for (uint32_t j0 = w * SW; j0 < (w + 1) * SW; j0 += 32) {
      const uint32_t k = ckeys[j0 + lane];
      const bool keep = !(k & kPurge);
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
      if (keep) *cnbr_out(J, base, X.a0, X.na, X.b0, wpos + __popc(bal & lt)) = k;
      wpos += __popc(bal);
      if (k != kEmpty) ckeys[j0 + lane] = kEmpty;
    }
    __syncthreads();
  }
}

__global__ void k_chub_finish(CHubJob H) {
  const uint32_t total = *H.list_count;
  uint32_t done = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    if (H.hk[i] == 0) continue;
    H.J.cnt[H.list[i]] = H.hcnt[i];
    ++done;
  }
  done = warp_sum(done);
  if (lane_id() == 0 && done) tier_add(H.J.tiers, HGP_TIER_CNBRS_H, done);
}

static constexpr uint32_t kCALog = 12, kCAThreads = 256;   // 4096 slots: 16 KB, <= 2048 entries
static constexpr uint32_t kCA2Log = 13;                     // 8192 slots: 32 KB, <= 4096 entries (5 CTAs/SM)
static constexpr uint32_t kCMLog = 14, kCMThreads = 256;   // 16384 slots: 64 KB, <= 8192 entries (3 CTAs/SM)
static constexpr uint32_t kCBLog = 15, kCBThreads = 256;   // 32768 slots: 128 KB, <= 16384 entries

static uint32_t grid_n(hgp_ctx *c, uint64_t n, uint32_t per = 256) {
  const uint64_t b = (n + per - 1) / per, cap = 16ull * c->sm_count;
  return (uint32_t)(b < cap ? (b ? b : 1) : cap);
}

// gamma (reading #11): coarse id = rank of the cluster's min member; coarse sizes;
// members mem0 (min) / mem1 (partner or NONE) of every coarse node. mem may be nullptr.
static hgp_status gamma_impl(hgp_ctx *c, const uint32_t *match, uint32_t N, const uint32_t *node_w, uint32_t *gamma,
                             uint32_t *Nc_out, uint32_t **cw_out, uint32_t **mem_out, bool cw_device_owned) {
  hgp_status st = HGP_OK;
  uint32_t *rep = scratch_raw<uint32_t>(c, N, &st);
  uint64_t *cid = scratch_raw<uint64_t>(c, (size_t)N + 1, &st);
  if (st) return st;
  HGP_TRY(clear_errors(c));
  HGP_TRY(launch(c, "rep", k_rep, dim3(grid_n(c, N)), dim3(256), 0, match, N, rep, c->d_err));
  uint64_t Nc64 = 0;
  HGP_TRY(scan_exclusive(c, InU32{rep}, N, cid, &Nc64));
  uint64_t err[kErrSlots];
  HGP_TRY(fetch_errors(c, err));
  if (err[kErrMatch] != UINT64_MAX)
    return set_error(HGP_E_ARG, "node %llu: match is not symmetric", (unsigned long long)err[kErrMatch]);
  const uint32_t Nc = (uint32_t)Nc64;
  uint32_t *cw = !node_w ? nullptr : cw_device_owned ? dalloc_n<uint32_t>(c, Nc, &st) : scratch_raw<uint32_t>(c, Nc, &st);
  uint32_t *mem = scratch_raw<uint32_t>(c, 2 * (size_t)Nc, &st);
  if (st) return st;
  if (cw) HGP_CUDA(cudaMemsetAsync(cw, 0, 4 * (size_t)(Nc ? Nc : 1), c->stream));
  HGP_TRY(launch(c, "gamma", k_gamma, dim3(grid_n(c, N)), dim3(256), 0, match, (const uint64_t *)cid, node_w, N,
                 gamma, cw, mem, mem + Nc));
  *Nc_out = Nc;
  if (cw_out) *cw_out = cw;
  if (mem_out) *mem_out = mem;
  return HGP_OK;
}

// Coarse edges of the fine edges [elo, ehi) before the merge (reading #13-14): pins
// mapped by gamma into the range's own oversized slots x[edge_off[e] - edge_off[elo] ..], src and
// dst blocks sorted, S' = unique src \ D', D' = unique dst, kept unless D' = ∅ and |S'| <= 1, and
// the 64-bit fingerprint of (|S'|, S', D').
struct EdgeRange {
  uint32_t *x, *cnsrc, *csize;
  uint8_t *keep;
  uint64_t *fp;
  const uint64_t *off;     // [n+1] offsets of the range's slots in x (relative)
  uint32_t n;
};

__global__ void k_rel_off(const uint64_t *edge_off, uint32_t elo, uint32_t n, uint64_t *rel) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    rel[i] = edge_off[elo + i] - edge_off[elo];
}

__global__ void k_cedges_pack(EdgeRange R, uint32_t elo, const uint64_t *pos, const uint64_t *poff, uint32_t *eid,
                              uint64_t *fp, uint32_t *nsrc, uint32_t *size, uint64_t *off, uint32_t *pins) {
  const uint32_t lane = lane_id();
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < R.n; i += nw) {
    if (!R.keep[i]) continue;
    const uint64_t k = pos[i], o = poff[i];
    const uint32_t n = R.csize[i];
    if (lane == 0) {
      eid[k] = elo + (uint32_t)i; fp[k] = R.fp[i]; nsrc[k] = R.cnsrc[i]; size[k] = n; off[k] = o;
    }
    const uint32_t *src = R.x + R.off[i];
    for (uint32_t j = lane; j < n; j += 32) pins[o + j] = src[j];
  }
}
struct KeptFlag {
  const uint8_t *keep;
  __device__ uint64_t operator()(uint64_t i) const { return keep[i]; }
};
struct KeptSize {
  const uint8_t *keep;
  const uint32_t *size;
  __device__ uint64_t operator()(uint64_t i) const { return keep[i] ? size[i] : 0u; }
};

static hgp_status edges_impl(hgp_ctx *c, const hgp_csr *g, const uint32_t *gamma, uint32_t elo, uint32_t ehi,
                             EdgeRange *R) {
  hgp_status st = HGP_OK;
  const uint32_t n = ehi - elo;
  uint64_t p0 = 0, p1 = 0;
  if (elo == 0 && ehi == g->E) {
    p1 = g->P;
  } else {
    uint64_t b[2];
    HGP_TRY(read_back(c, g->edge_off + elo, 8, &b[0]));
    HGP_TRY(read_back(c, g->edge_off + ehi, 8, &b[1]));
    p0 = b[0];
    p1 = b[1];
  }
  const uint64_t Pr = p1 - p0;
  R->n = n;
  R->x = scratch_raw<uint32_t>(c, Pr, &st);
  R->cnsrc = scratch_raw<uint32_t>(c, n, &st);
  R->csize = scratch_raw<uint32_t>(c, n, &st);
  R->keep = scratch_raw<uint8_t>(c, n, &st);
  R->fp = scratch_raw<uint64_t>(c, n, &st);
  if (st) return st;
  if (elo == 0) {
    R->off = g->edge_off;                                           // p0 = 0: fine offsets are relative
  } else {
    uint64_t *rel = scratch_raw<uint64_t>(c, (size_t)n + 1, &st);
    if (st) return st;
    HGP_TRY(launch(c, "rel_off", k_rel_off, dim3(grid_n(c, (uint64_t)n + 1)), dim3(256), 0,
                   (const uint64_t *)g->edge_off, elo, n, rel));
    R->off = rel;
  }
  if (n == 0) return HGP_OK;
  HGP_TRY(launch(c, "map_pins", k_map_pins, dim3(grid_n(c, Pr)), dim3(256), 0, (const uint32_t *)g->pins + p0,
                 gamma, Pr, R->x));
  HGP_TRY(segmented_sort(c, EdgeSeg2{R->off, g->edge_nsrc + elo}, 2 * (uint64_t)n, R->x, g->max_edge));
  HGP_TRY(launch(c, "edge_unique", k_edge_unique, dim3(grid_n(c, n, 8)), dim3(256), 0, R->off,
                 (const uint32_t *)g->edge_nsrc + elo, n, R->x, R->cnsrc, R->csize, R->keep, R->fp));
  return HGP_OK;
}

// Merge of the entries of M (identical (S', D') -> one coarse edge, omega' = sum, mu' = sum,
// ordered by the minimum fine id; reading #12) into C's edge arrays and incidence.
static hgp_status merge_impl(hgp_ctx *c, const hgp_csr *g, MergeJob M, hgp_csr *C, uint32_t *erep_out) {
  hgp_status st = HGP_OK;
  const uint32_t K = M.E;
  uint32_t log2t = 4;
  while ((1ull << log2t) < 2ull * K + 16) ++log2t;
  M.owner = scratch_raw<uint32_t>(c, (size_t)1 << log2t, &st);
  M.minrep = scratch_raw<uint32_t>(c, (size_t)1 << log2t, &st);
  M.slot_of = scratch_raw<uint32_t>(c, K, &st);
  M.log2t = log2t;
  uint32_t *erep = erep_out ? erep_out : scratch_raw<uint32_t>(c, K, &st);
  uint32_t *is_rep = scratch_raw<uint32_t>(c, K, &st);
  uint64_t *ceid = scratch_raw<uint64_t>(c, (size_t)K + 1, &st);
  if (st) return st;
  HGP_CUDA(cudaMemsetAsync(M.owner, 0xFF, 4ull << log2t, c->stream));
  HGP_CUDA(cudaMemsetAsync(M.minrep, 0xFF, 4ull << log2t, c->stream));
  HGP_TRY(launch(c, "merge_insert", k_merge_insert, dim3(grid_n(c, K)), dim3(256), 0, M));
  HGP_TRY(launch(c, "merge_resolve", k_merge_resolve, dim3(grid_n(c, K)), dim3(256), 0, M, erep, is_rep));
  uint64_t Ec64 = 0;
  HGP_TRY(scan_exclusive(c, InU32{is_rep}, K, ceid, &Ec64));
  const uint32_t Ec = (uint32_t)Ec64;
  C->E = Ec;
  C->edge_off = dalloc_n<uint64_t>(c, (size_t)Ec + 1, &st);
  C->edge_nsrc = dalloc_n<uint32_t>(c, Ec, &st);
  C->edge_w = dalloc_n<uint32_t>(c, Ec, &st);
  C->edge_mu = dalloc_n<uint32_t>(c, Ec, &st);
  uint32_t *c_size = scratch_raw<uint32_t>(c, Ec, &st);
  unsigned int *maxes = scratch_zero<unsigned int>(c, 4, &st);
  if (st) return st;
  HGP_CUDA(cudaMemsetAsync(C->edge_w, 0, 4 * (size_t)(Ec ? Ec : 1), c->stream));
  HGP_CUDA(cudaMemsetAsync(C->edge_mu, 0, 4 * (size_t)(Ec ? Ec : 1), c->stream));
  HGP_TRY(launch(c, "coarse_edge_attrs", k_coarse_edge_attrs, dim3(grid_n(c, K)), dim3(256), 0, (const uint32_t *)erep,
                 (const uint64_t *)ceid, (const uint32_t *)g->edge_w, (const uint32_t *)g->edge_mu, M.cnsrc, M.csize, K,
                 M.eid, C->edge_w, C->edge_mu, C->edge_nsrc, c_size));
  uint64_t Pc = 0;
  HGP_TRY(scan_exclusive(c, InU32{c_size}, Ec, C->edge_off, &Pc));
  C->P = Pc;
  C->pins = dalloc_n<uint32_t>(c, Pc, &st);
  if (st) return st;
  HGP_TRY(launch(c, "coarse_edge_pack", k_coarse_edge_pack, dim3(grid_n(c, K, 8)), dim3(256), 0, (const uint32_t *)erep,
                 (const uint64_t *)ceid, M.off, M.x, M.csize, (const uint64_t *)C->edge_off, K, C->pins, maxes));
  uint32_t hmax[4];
  HGP_TRY(read_back(c, maxes, 16, hmax));
  C->max_edge = hmax[0];
  return build_incidence(c, C);
}

// Coarse neighbours (reading #7, #16) of the coarse nodes [clo, chi): member
// segments are read through J's view (nb_off or nb_start/nb_len over nbr).
static hgp_status cnbrs_impl(hgp_ctx *c, CNbrJob J, uint32_t clo, uint32_t chi, hgp_nbrs *CN, uint64_t *purged_out,
                             bool inplace = false) {
  hgp_status st = HGP_OK;
  const uint32_t Nc = chi - clo;
  // the kernels index coarse nodes from 0: shift the member arrays
  J.mem0 += clo;
  J.mem1 += clo;
  uint64_t *bound_off = scratch_raw<uint64_t>(c, (size_t)Nc + 1, &st);
  if (st) return st;
  uint64_t Vb = 0;
  HGP_TRY(scan_exclusive(c, BoundIn{J.mem0, J.mem1, J.nb_off, J.nb_off ? nullptr : J.nb_len}, Nc, bound_off, &Vb));
  // in place (the level-0 pool view, consumed by this call): no bound pool — N'(c) overwrites the
  // segments of its members (C5: saves V entries, ~40 GB)
  uint32_t *pool = inplace ? nullptr : scratch_raw<uint32_t>(c, Vb, &st);
  uint32_t *ccnt = scratch_raw<uint32_t>(c, Nc, &st);
  uint32_t *lists = scratch_raw<uint32_t>(c, 4 * (size_t)Nc, &st);   // M, B, C, A2
  uint32_t *counts = scratch_zero<uint32_t>(c, 4, &st);
  unsigned long long *misc = scratch_zero<unsigned long long>(c, 2, &st);   // purged, max bound (tier C)
  unsigned int *maxes = scratch_zero<unsigned int>(c, 2, &st);
  if (st) return st;
  static uint64_t attr_dev = 0;   // per device: cudaFuncSetAttribute applies to the current one
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_coarse_nbrs<kCAThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 << kCALog);
    // tiers M and B share the instantiation <256, true>: the attribute is the larger table's
    static_assert(kCMThreads == kCBThreads && kCMLog < kCBLog, "M and B share one instantiation");
    cudaFuncSetAttribute(k_coarse_nbrs<kCBThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 << kCBLog);
  }
  J.bound_off = bound_off;
  J.pool = pool; J.cnt = ccnt; J.Nc = Nc; J.purged = misc; J.tiers = c->d_tiers; J.tier = HGP_TIER_CNBRS_A;
  J.nbr_w = inplace ? const_cast<uint32_t *>(J.nbr) : nullptr;
  J.cbase = clo;
  const uint32_t capA = 1u << (kCALog - 1), capA2 = 1u << (kCA2Log - 1), capM = 1u << (kCMLog - 1), capB = 1u << (kCBLog - 1);
  J.list = nullptr; J.list_count = nullptr; J.cap = capA; J.log2s = kCALog;
  const uint32_t gA = Nc < 64u * c->sm_count ? (Nc ? Nc : 1) : 64u * c->sm_count;
  if (Nc) HGP_TRY(launch(c, "coarse_nbrs_A", k_coarse_nbrs<kCAThreads, true>, dim3(gA), dim3(kCAThreads), 5u << kCALog, J));
  if (Nc) HGP_TRY(launch(c, "cnbr_classify", k_cnbr_classify, dim3(grid_n(c, Nc)), dim3(256), 0, (const uint64_t *)bound_off,
                         Nc, capA, capA2, capM, capB, lists + 3 * (size_t)Nc, lists, lists + Nc, lists + 2 * (size_t)Nc,
                         counts, misc + 1));
  uint32_t hc[4];
  HGP_TRY(read_back(c, counts, 16, hc));
  if (hc[3]) {   // between A and M: 40 KB, 5 CTAs/SM (M's 80 KB tables allow 2)
    J.list = lists + 3 * (size_t)Nc; J.list_count = counts + 3; J.cap = capA2; J.log2s = kCA2Log; J.tier = HGP_TIER_CNBRS_A2;
    const uint32_t g2 = resident_grid(c, k_coarse_nbrs<kCMThreads, true>, kCMThreads, 5u << kCA2Log);
    HGP_TRY(launch(c, "coarse_nbrs_A2", k_coarse_nbrs<kCMThreads, true>, dim3(g2), dim3(kCMThreads), 5u << kCA2Log, J));
  }
  if (hc[0]) {
    J.list = lists; J.list_count = counts; J.cap = capM; J.log2s = kCMLog; J.tier = HGP_TIER_CNBRS_M;
    HGP_TRY(launch(c, "coarse_nbrs_M", k_coarse_nbrs<kCMThreads, true>, dim3(2 * c->sm_count), dim3(kCMThreads),
                   5u << kCMLog, J));
  }
  if (hc[1]) {
    J.list = lists + Nc; J.list_count = counts + 1; J.cap = capB; J.log2s = kCBLog; J.tier = HGP_TIER_CNBRS_B;
    HGP_TRY(launch(c, "coarse_nbrs_B", k_coarse_nbrs<kCBThreads, true>, dim3(c->sm_count), dim3(kCBThreads),
                   5u << kCBLog, J));
  }
  uint32_t *listC = lists + 2 * (size_t)Nc, *countC = counts + 2;
  if (hc[2] && !c->opt.no_hub) {   // hubs: key-partitioned shared tables; what they leave -> tier C
    const uint32_t hn = hc[2];
    CHubJob H{};
    H.J = J;
    H.list = listC; H.list_count = countC;
    H.hk = scratch_raw<uint32_t>(c, hn, &st);
    H.hb = scratch_raw<uint64_t>(c, hn, &st);
    H.hcnt = scratch_raw<uint32_t>(c, hn, &st);
    uint64_t *item_off = scratch_raw<uint64_t>(c, (size_t)hn + 1, &st);
    uint64_t *vis_off = scratch_raw<uint64_t>(c, (size_t)hn + 1, &st);
    H.lu = scratch_raw<uint32_t>(c, hn, &st);
    H.lu_count = scratch_zero<uint32_t>(c, 1, &st);
    if (st) return st;
    H.item_off = item_off; H.vis_off = vis_off;
    const uint32_t gh = hn < 4u * c->sm_count ? hn : 4u * c->sm_count;
    HGP_TRY(launch(c, "chub_size", k_chub_visit<0>, dim3(gh), dim3(kCHThreads), 0, H));
    uint64_t nitems = 0, nvis = 0;
    HGP_TRY(scan_exclusive(c, InU32{H.hk}, hn, item_off, &nitems));
    HGP_TRY(scan_exclusive(c, InU64{H.hb}, hn, vis_off, &nvis));
    if (nitems > 0xFFFFFFFFull) return set_error(HGP_E_OVERFLOW, "coarse hub tier: too many partitions");
    if (nitems) {
      H.ibase = scratch_raw<uint32_t>(c, nitems, &st);
      H.ilen = scratch_raw<uint32_t>(c, nitems, &st);
      H.inode = scratch_raw<uint32_t>(c, nitems, &st);
      H.bkey = scratch_raw<uint32_t>(c, nvis, &st);
      if (st) return st;
      HGP_TRY(launch(c, "chub_scatter", k_chub_visit<1>, dim3(gh), dim3(kCHThreads), 0, H));
      const size_t smem = 4u << kCHLog;
      const uint32_t gi0 = resident_grid(c, k_chub_items, kCHThreads, smem);
      HGP_TRY(launch(c, "chub_items", k_chub_items, dim3(nitems < gi0 ? (uint32_t)nitems : gi0), dim3(kCHThreads), smem, H,
                     (uint32_t)nitems));
      HGP_TRY(launch(c, "chub_finish", k_chub_finish, dim3(grid_n(c, hn)), dim3(256), 0, H));
    }
    HGP_TRY(read_back(c, H.lu_count, 4, &hc[2]));
    listC = H.lu; countC = H.lu_count;
  }
  if (hc[2]) {
    uint64_t mb = 0;
    if (listC != lists + 2 * (size_t)Nc) {   // the hub tier's leftovers: their own max bound
      HGP_CUDA(cudaMemsetAsync(misc + 1, 0, 8, c->stream));
      HGP_TRY(launch(c, "cnbr_maxb", k_list_max_bound, dim3(grid_n(c, hc[2])), dim3(256), 0, (const uint64_t *)bound_off,
                     (const uint32_t *)listC, (const uint32_t *)countC, misc + 1));
    }
    HGP_TRY(read_u64(c, (const uint64_t *)(misc + 1), &mb));
    uint32_t lg = kCBLog;
    while ((1ull << (lg - 1)) < mb) ++lg;
    const uint32_t ctas = hc[2] < (uint32_t)c->sm_count ? hc[2] : (uint32_t)c->sm_count;
    uint32_t *gtab = scratch_raw<uint32_t>(c, (size_t)ctas << lg, &st);
    if (st) return st;
    J.list = listC; J.list_count = countC; J.cap = 0xFFFFFFFFu; J.log2s = lg; J.gtab = gtab;
    J.tier = HGP_TIER_CNBRS_C;
    HGP_TRY(launch(c, "coarse_nbrs_C", k_coarse_nbrs<256, false>, dim3(ctas), dim3(256), 0, J));
  }
  CN->lo = clo;
  CN->hi = chi;
  CN->off = dalloc_n<uint64_t>(c, (size_t)Nc + 1, &st);
  if (st) return st;
  uint64_t Vc = 0;
  HGP_TRY(scan_exclusive(c, InU32{ccnt}, Nc, CN->off, &Vc));
  CN->V = Vc;
  CN->nbr = dalloc_n<uint32_t>(c, Vc, &st);
  if (st) return st;
  if (Nc && !inplace)
    HGP_TRY(launch(c, "cnbr_pack", k_cnbr_pack_flat<false>, dim3(8u * c->sm_count), dim3(256), 0, J, (const uint32_t *)pool,
                   (const uint64_t *)bound_off, (const uint64_t *)CN->off, Nc, Vc, CN->nbr, maxes));
  if (Nc && inplace)
    HGP_TRY(launch(c, "cnbr_pack", k_cnbr_pack_flat<true>, dim3(8u * c->sm_count), dim3(256), 0, J, (const uint32_t *)nullptr,
                   (const uint64_t *)nullptr, (const uint64_t *)CN->off, Nc, Vc, CN->nbr, maxes));
  uint32_t hmax[2];
  HGP_TRY(read_back(c, maxes, 8, hmax));
  CN->max_deg = hmax[0];
  if (purged_out) HGP_TRY(read_u64(c, (const uint64_t *)misc, purged_out));
  return HGP_OK;
}

hgp_status contract_impl(hgp_ctx *c, const hgp_csr *g, const hgp_nbrs *nb, const uint32_t *match, uint32_t *gamma,
                         hgp_csr *C, hgp_nbrs *CN, hgp_level_stats *stats, const SegView *view) {
  hgp_status st = HGP_OK;
  const uint32_t N = g->N, E = g->E;
  memset(C, 0, sizeof(*C));
  memset(CN, 0, sizeof(*CN));
  uint32_t Nc = 0, *mem = nullptr;
  HGP_TRY(gamma_impl(c, match, N, g->node_w, gamma, &Nc, &C->node_w, &mem, true));
  C->N = Nc;
  EdgeRange R{};
  HGP_TRY(edges_impl(c, g, gamma, 0, E, &R));
  MergeJob M{};
  M.off = R.off; M.x = R.x; M.cnsrc = R.cnsrc; M.csize = R.csize; M.keep = R.keep; M.fp = R.fp; M.eid = nullptr;
  M.E = E;
  uint32_t *erep = scratch_raw<uint32_t>(c, E, &st);
  if (st) return st;
  HGP_TRY(merge_impl(c, g, M, C, erep));
  CNbrJob J{};
  J.mem0 = mem; J.mem1 = mem + Nc; J.gamma = gamma;
  J.nb_off = view ? nullptr : nb->off;
  J.nb_start = view ? view->start : nullptr; J.nb_len = view ? view->len : nullptr;
  J.nbr = view ? view->nbr : nb->nbr;
  uint64_t purged = 0;
  HGP_TRY(cnbrs_impl(c, J, 0, Nc, CN, &purged, view != nullptr));
  if (stats) {
    // kept edges = classes' members; dropped = E - kept; merged = kept - Ec
    uint32_t *kc = scratch_zero<uint32_t>(c, 1, &st);
    if (st) return st;
    HGP_TRY(launch(c, "count_kept", k_count_kept, dim3(grid_n(c, E)), dim3(256), 0, (const uint32_t *)erep, E, kc));
    uint32_t hk = 0;
    HGP_TRY(read_back(c, kc, 4, &hk));
    stats->Nc = Nc; stats->Ec = C->E; stats->Pc = C->P; stats->Vc = CN->V;
    stats->dropped_edges = (uint32_t)(E - hk);
    stats->merged_edges = (uint32_t)(hk - C->E);
    stats->purged = purged;
  }
  return HGP_OK;
}

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_contract(hgp_ctx *c, const hgp_csr *g, const hgp_nbrs *nb, const uint32_t *match,
                                   uint32_t *gamma, hgp_csr *coarse, hgp_nbrs *coarse_nb) {
  if (!c || !g || !nb || !match || !gamma || !coarse || !coarse_nb)
    return set_error(HGP_E_ARG, "hgp_contract: null argument");
  if (nb->lo != 0 || nb->hi != g->N) return set_error(HGP_E_ARG, "contract needs neighbours of every node");
  ApiScope scope(c);
  hgp_status s = contract_impl(c, g, nb, match, gamma, coarse, coarse_nb, nullptr, nullptr);
  if (s != HGP_OK) { free_csr(c, coarse); free_nbrs(c, coarse_nb); }
  return s;
}

// ---- a5 in pieces for node/edge-range shards; hgp_contract = these on one GPU.
extern "C" {

__global__ void k_coarse_bounds(const uint64_t *cid, const uint32_t *nb, uint32_t nbounds, uint64_t *cb) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nbounds; i += gridDim.x * blockDim.x) cb[i] = cid[nb[i]];
}

hgp_status hgp_coarse_bounds(hgp_ctx *c, const uint32_t *match, uint32_t N, const uint32_t *node_bounds, uint32_t nbounds,
                             uint32_t *coarse_bounds) {
  if (!c || (N && !match) || !node_bounds || !coarse_bounds) return set_error(HGP_E_ARG, "hgp_coarse_bounds: null argument");
  ApiScope scope(c);
  hgp_status st = HGP_OK;
  uint32_t *rep = scratch_raw<uint32_t>(c, N, &st);
  uint64_t *cid = scratch_raw<uint64_t>(c, (size_t)N + 1, &st);
  uint32_t *db = scratch_raw<uint32_t>(c, nbounds, &st);
  uint64_t *dc = scratch_raw<uint64_t>(c, nbounds, &st);
  if (st) return st;
  for (uint32_t i = 0; i < nbounds; ++i)
    if (node_bounds[i] > N) return set_error(HGP_E_ARG, "hgp_coarse_bounds: bound %u > N", node_bounds[i]);
  HGP_TRY(clear_errors(c));
  HGP_TRY(launch(c, "rep", k_rep, dim3(grid_n(c, N)), dim3(256), 0, match, N, rep, c->d_err));
  HGP_TRY(scan_exclusive(c, InU32{rep}, N, cid, nullptr));
  HGP_CUDA(cudaMemcpyAsync(db, node_bounds, 4ull * nbounds, cudaMemcpyHostToDevice, c->stream));
  HGP_TRY(launch(c, "coarse_bounds", k_coarse_bounds, dim3(1), dim3(256), 0, (const uint64_t *)cid, (const uint32_t *)db,
                 nbounds, dc));
  std::vector<uint64_t> h(nbounds);
  HGP_TRY(read_back(c, dc, 8ull * nbounds, h.data()));
  for (uint32_t i = 0; i < nbounds; ++i) coarse_bounds[i] = (uint32_t)h[i];
  return HGP_OK;
}

hgp_status hgp_gamma(hgp_ctx *c, const uint32_t *match, uint32_t N, uint32_t *gamma, uint32_t *Nc) {
  if (!c || (N && (!match || !gamma)) || !Nc) return set_error(HGP_E_ARG, "hgp_gamma: null argument");
  ApiScope scope(c);
  return gamma_impl(c, match, N, nullptr, gamma, Nc, nullptr, nullptr, false);
}

void hgp_cedges_free(hgp_ctx *c, hgp_cedges *ce) {
  if (!c || !ce) return;
  DeviceGuard dg(c->device);
  const size_t K = ce->K ? ce->K : 1;
  c->dfree(ce->eid, 4 * K);
  c->dfree(ce->fp, 8 * K);
  c->dfree(ce->nsrc, 4 * K);
  c->dfree(ce->size, 4 * K);
  c->dfree(ce->off, 8 * (K + 1));
  c->dfree(ce->pins, 4 * (ce->P ? ce->P : 1));
  memset(ce, 0, sizeof(*ce));
}

hgp_status hgp_contract_edges(hgp_ctx *c, const hgp_csr *g, const uint32_t *gamma, uint32_t elo, uint32_t ehi,
                              hgp_cedges *out) {
  if (!c || !g || !gamma || !out) return set_error(HGP_E_ARG, "hgp_contract_edges: null argument");
  if (elo > ehi || ehi > g->E) return set_error(HGP_E_ARG, "hgp_contract_edges: bad edge range");
  ApiScope scope(c);
  memset(out, 0, sizeof(*out));
  hgp_status st = HGP_OK;
  EdgeRange R{};
  HGP_TRY(edges_impl(c, g, gamma, elo, ehi, &R));
  const uint32_t n = ehi - elo;
  uint64_t *pos = scratch_raw<uint64_t>(c, (size_t)n + 1, &st);
  uint64_t *poff = scratch_raw<uint64_t>(c, (size_t)n + 1, &st);
  if (st) return st;
  uint64_t K = 0, P = 0;
  HGP_TRY(scan_exclusive(c, KeptFlag{R.keep}, n, pos, &K));
  HGP_TRY(scan_exclusive(c, KeptSize{R.keep, R.csize}, n, poff, &P));
  out->K = (uint32_t)K;
  out->P = P;
  out->eid = dalloc_n<uint32_t>(c, K, &st);
  out->fp = dalloc_n<uint64_t>(c, K, &st);
  out->nsrc = dalloc_n<uint32_t>(c, K, &st);
  out->size = dalloc_n<uint32_t>(c, K, &st);
  out->off = dalloc_n<uint64_t>(c, K + 1, &st);
  out->pins = dalloc_n<uint32_t>(c, P, &st);
  if (st) { hgp_cedges_free(c, out); return st; }
  hgp_status s = HGP_OK;
  if (n)
    s = launch(c, "cedges_pack", k_cedges_pack, dim3(grid_n(c, (uint64_t)n * 32)), dim3(256), 0, R, elo,
               (const uint64_t *)pos, (const uint64_t *)poff, out->eid, out->fp, out->nsrc, out->size, out->off,
               out->pins);
  if (s == HGP_OK) s = hgp_copy(c, out->off + K, &P, 8) == HGP_OK ? hgp_sync(c) : HGP_E_CUDA;
  if (s != HGP_OK) hgp_cedges_free(c, out);
  return s;
}

hgp_status hgp_contract_merge(hgp_ctx *c, const hgp_csr *g, const uint32_t *match, uint32_t *gamma,
                              const hgp_cedges *all, hgp_csr *coarse) {
  if (!c || !g || !match || !gamma || !all || !coarse) return set_error(HGP_E_ARG, "hgp_contract_merge: null argument");
  ApiScope scope(c);
  memset(coarse, 0, sizeof(*coarse));
  uint32_t Nc = 0;
  hgp_status s = gamma_impl(c, match, g->N, g->node_w, gamma, &Nc, &coarse->node_w, nullptr, true);
  if (s == HGP_OK) {
    coarse->N = Nc;
    MergeJob M{};
    M.off = all->off; M.x = all->pins; M.cnsrc = all->nsrc; M.csize = all->size; M.keep = nullptr; M.fp = all->fp;
    M.eid = all->eid; M.E = all->K;
    s = merge_impl(c, g, M, coarse, nullptr);
  }
  if (s != HGP_OK) free_csr(c, coarse);
  return s;
}

hgp_status hgp_coarse_neighbors(hgp_ctx *c, const uint32_t *match, const uint32_t *gamma, uint32_t N,
                                const uint64_t *seg_start, const uint32_t *seg_len, const uint32_t *nbr, uint32_t clo,
                                uint32_t chi, hgp_nbrs *out) {
  if (!c || !match || !gamma || !seg_start || !seg_len || !out) return set_error(HGP_E_ARG, "hgp_coarse_neighbors: null argument");
  ApiScope scope(c);
  memset(out, 0, sizeof(*out));
  uint32_t Nc = 0, *mem = nullptr;
  // the members of every coarse node (gamma is recomputed, identically, into scratch)
  hgp_status st = HGP_OK;
  uint32_t *g2 = scratch_raw<uint32_t>(c, N, &st);
  if (st) return st;
  hgp_status s = gamma_impl(c, match, N, nullptr, g2, &Nc, nullptr, &mem, false);
  if (s != HGP_OK) return s;
  if (clo > chi || chi > Nc) return set_error(HGP_E_ARG, "hgp_coarse_neighbors: bad coarse range");
  CNbrJob J{};
  J.mem0 = mem; J.mem1 = mem + Nc; J.gamma = gamma;
  J.nb_off = nullptr; J.nb_start = seg_start; J.nb_len = seg_len; J.nbr = nbr;
  s = cnbrs_impl(c, J, clo, chi, out, nullptr);
  if (s != HGP_OK) free_nbrs(c, out);
  return s;
}

}  // extern "C"
