// lbs.cuh — load-balanced search: pin-parallel iteration over a CSR of hyperedges.
// A CTA owns a tile of consecutive pins; it stages the offsets of the edges overlapping
// the tile in shared memory and every thread finds its pin's edge by a short binary
// search there. Full lane utilisation whatever the edge-size distribution (C3: |e| = 2..1024).
#pragma once
#include "common.cuh"

namespace hgp {

constexpr int kLbsThreads = 256;
constexpr int kLbsItems = 8;
constexpr int kLbsTile = kLbsThreads * kLbsItems;

// first index i in [0, n) with a[i] > x (n if none)
__device__ __forceinline__ uint32_t upper_bound_u64(const uint64_t *a, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct LbsShared {
  uint64_t off[kLbsTile + 2];
  uint32_t e0, ne;      // edges e0 .. e0+ne-1 overlap the tile; ne == 0xFFFFFFFF: use global search
};

// Stage the tile [p0, p0 + kLbsTile) ∩ [0, P). Must be called by all threads of the CTA.
__device__ __forceinline__ void lbs_stage(LbsShared &sh, const uint64_t *edge_off, uint32_t E, uint64_t p0,
                                          uint64_t P) {
  if (threadIdx.x == 0) {
    uint64_t plast = p0 + kLbsTile - 1 < P ? p0 + kLbsTile - 1 : P - 1;
    uint32_t a = upper_bound_u64(edge_off, E + 1, p0) - 1;
    uint32_t b = upper_bound_u64(edge_off, E + 1, plast) - 1;
    sh.e0 = a;
    sh.ne = (b - a + 1 <= (uint32_t)kLbsTile + 1) ? b - a + 1 : 0xFFFFFFFFu;
  }
  __syncthreads();
  if (sh.ne != 0xFFFFFFFFu)
    for (uint32_t k = threadIdx.x; k <= sh.ne; k += blockDim.x) sh.off[k] = edge_off[sh.e0 + k];
  __syncthreads();
}

// edge containing pin p (p inside the staged tile)
__device__ __forceinline__ uint32_t lbs_edge(const LbsShared &sh, const uint64_t *edge_off, uint32_t E, uint64_t p) {
  if (sh.ne == 0xFFFFFFFFu) return upper_bound_u64(edge_off, E + 1, p) - 1;
  uint32_t lo = 0, hi = sh.ne + 1;   // search sh.off[0..ne]
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (sh.off[mid] <= p) lo = mid + 1; else hi = mid;
  }
  return sh.e0 + lo - 1;
}

}  // namespace hgp
