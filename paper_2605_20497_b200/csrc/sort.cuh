// sort.cuh — CUB-free segmented sort of u32 keys for small/medium segments.
//
// Tiers: len <= 32 register bitonic (one warp); len <= kWarpSortCap smem bitonic by one
// warp; len <= kCtaSortCap smem bitonic by one CTA; larger: bitonic in global memory by
// one CTA. The bitonic network is the "flip" form, which sorts any length n when the
// virtual tail [n, next_pow2(n)) is +inf: compare-exchanges that touch the tail are no-ops.
#pragma once
#include "common.cuh"

namespace hgp {

constexpr uint32_t kWarpSortCap = 1024;
constexpr uint32_t kCtaSortCap = 16384;
constexpr int kSortWarpsPerCta = 8;
constexpr int kCtaSortThreads = 512;

__device__ __forceinline__ uint32_t next_pow2(uint32_t n) { return n <= 1 ? 1 : 1u << (32 - __clz(n - 1)); }

// Sort 32 lanes' keys ascending (lanes >= len must hold 0xFFFFFFFF).
__device__ __forceinline__ uint32_t warp_bitonic32(uint32_t key) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, key, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      uint32_t mn = min(key, other), mx = max(key, other);
      key = (lower == up) ? mn : mx;
    }
  }
  return key;
}

// Sort up to 128 keys held 4 per lane (element index i*32 + lane); padding must be 0xFFFFFFFF.
// Classic bitonic network: stages with j >= 32 pair registers of the same lane, j < 32 pair lanes.
__device__ __forceinline__ void warp_bitonic128(uint32_t (&v)[4]) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (uint32_t k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const uint32_t d = j >> 5;
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) {
          if (i & d) continue;
          const uint32_t x = i * 32 + lane;                 // lower index of the pair (i, i|d)
          const bool up = (x & k) == 0;
          const uint32_t a = v[i], b = v[i | d];
          const uint32_t mn = min(a, b), mx = max(a, b);
          v[i] = up ? mn : mx;
          v[i | d] = up ? mx : mn;
        }
      } else {
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) {
          const uint32_t x = i * 32 + lane;
          const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, v[i], j);
          const bool up = (x & k) == 0;
          const bool lower = (lane & j) == 0;
          const uint32_t mn = min(v[i], other), mx = max(v[i], other);
          v[i] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// Sort s[0..n) ascending with nthreads cooperating threads (index tid); SYNC is the barrier.
template <class Sync>
__device__ __forceinline__ void bitonic_sort_flip(uint32_t *s, uint32_t n, uint32_t tid, uint32_t nthreads,
                                                  Sync sync) {
  const uint32_t N2 = next_pow2(n), half_total = N2 >> 1;
  for (uint32_t k = 2; k <= N2; k <<= 1) {
    const uint32_t h = k >> 1, lh = __ffs(h) - 1;
    for (uint32_t i = tid; i < half_total; i += nthreads) {
      uint32_t blk = i >> lh, off = i & (h - 1);
      uint32_t a = blk * k + off, b = blk * k + k - 1 - off;
      if (b < n) {
        uint32_t x = s[a], y = s[b];
        if (x > y) { s[a] = y; s[b] = x; }
      }
    }
    sync();
    for (uint32_t j = k >> 2; j > 0; j >>= 1) {
      const uint32_t lj = __ffs(j) - 1;
      for (uint32_t i = tid; i < half_total; i += nthreads) {
        uint32_t a = ((i >> lj) << (lj + 1)) + (i & (j - 1)), b = a + j;
        if (b < n) {
          uint32_t x = s[a], y = s[b];
          if (x > y) { s[a] = y; s[b] = x; }
        }
      }
      sync();
    }
  }
}

struct WarpSync { __device__ void operator()() const { __syncwarp(); } };
struct CtaSync { __device__ void operator()() const { __syncthreads(); } };

// Segment descriptor functor: seg(i, &beg, &len).
template <class Seg>
__global__ void __launch_bounds__(kSortWarpsPerCta * 32)
k_segsort_warp(Seg seg, uint64_t nseg, uint32_t *keys, uint64_t *big, uint32_t *nbig) {
  __shared__ uint32_t buf[kSortWarpsPerCta][kWarpSortCap];
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint64_t gw = (uint64_t)blockIdx.x * kSortWarpsPerCta + w, nw = (uint64_t)gridDim.x * kSortWarpsPerCta;
  for (uint64_t i = gw; i < nseg; i += nw) {
    uint64_t beg;
    uint32_t len;
    seg(i, beg, len);
    if (len <= 1) continue;
    uint32_t *k = keys + beg;
    if (len <= 32) {
      uint32_t v = lane < len ? k[lane] : 0xFFFFFFFFu;
      v = warp_bitonic32(v);
      if (lane < len) k[lane] = v;
    } else if (len <= 128) {
      uint32_t v[4];
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i) v[i] = i * 32 + lane < len ? k[i * 32 + lane] : 0xFFFFFFFFu;
      warp_bitonic128(v);
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i)
        if (i * 32 + lane < len) k[i * 32 + lane] = v[i];
    } else if (len <= kWarpSortCap) {
      uint32_t *s = buf[w];
      for (uint32_t j = lane; j < len; j += 32) s[j] = k[j];
      __syncwarp();
      bitonic_sort_flip(s, len, lane, 32, WarpSync{});
      for (uint32_t j = lane; j < len; j += 32) k[j] = s[j];
      __syncwarp();
    } else if (lane == 0) {
      uint32_t slot = atomicAdd(nbig, 1u);
      big[slot] = i;
    }
  }
}

template <class Seg>
__global__ void __launch_bounds__(kCtaSortThreads)
k_segsort_cta(Seg seg, const uint64_t *big, const uint32_t *nbig, uint32_t *keys, uint64_t *huge,
              uint32_t *nhuge) {
  extern __shared__ uint32_t sbuf[];
  const uint32_t count = *nbig;
  for (uint32_t t = blockIdx.x; t < count; t += gridDim.x) {
    uint64_t beg;
    uint32_t len;
    seg(big[t], beg, len);
    if (len > kCtaSortCap) {
      if (threadIdx.x == 0) huge[atomicAdd(nhuge, 1u)] = big[t];
      continue;
    }
    uint32_t *k = keys + beg;
    for (uint32_t j = threadIdx.x; j < len; j += blockDim.x) sbuf[j] = k[j];
    __syncthreads();
    bitonic_sort_flip(sbuf, len, threadIdx.x, blockDim.x, CtaSync{});
    for (uint32_t j = threadIdx.x; j < len; j += blockDim.x) k[j] = sbuf[j];
    __syncthreads();
  }
}

template <class Seg>
__global__ void __launch_bounds__(1024)
k_segsort_global(Seg seg, const uint64_t *huge, const uint32_t *nhuge, uint32_t *keys) {
  const uint32_t count = *nhuge;
  for (uint32_t t = blockIdx.x; t < count; t += gridDim.x) {
    uint64_t beg;
    uint32_t len;
    seg(huge[t], beg, len);
    bitonic_sort_flip(keys + beg, len, threadIdx.x, blockDim.x, CtaSync{});
  }
}

// Sort every segment of `keys` ascending. Asynchronous (no host sync).
template <class Seg>
hgp_status segmented_sort(hgp_ctx *c, Seg seg, uint64_t nseg, uint32_t *keys, uint32_t max_len) {
  if (nseg == 0 || max_len <= 1) return HGP_OK;
  hgp_status st = HGP_OK;
  const uint32_t warps_needed = (uint32_t)((nseg + kSortWarpsPerCta - 1) / kSortWarpsPerCta);
  const uint32_t grid = warps_needed < 64u * c->sm_count ? warps_needed : 64u * c->sm_count;
  if (max_len <= kWarpSortCap) {
    return launch(c, "segsort_warp", k_segsort_warp<Seg>, dim3(grid), dim3(kSortWarpsPerCta * 32), 0, seg,
                  nseg, keys, (uint64_t *)nullptr, (uint32_t *)nullptr);
  }
  uint32_t *cnt = scratch_zero<uint32_t>(c, 2, &st);
  uint64_t *big = scratch_raw<uint64_t>(c, nseg, &st);
  uint64_t *huge = scratch_raw<uint64_t>(c, nseg, &st);
  if (st != HGP_OK) return st;
  HGP_TRY(launch(c, "segsort_warp", k_segsort_warp<Seg>, dim3(grid), dim3(kSortWarpsPerCta * 32), 0, seg, nseg,
                 keys, big, cnt));
  static uint64_t attr_dev = 0;
  if (once_per_device(&attr_dev, c->device)) {
    cudaFuncSetAttribute(k_segsort_cta<Seg>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSortCap * 4);
  }
  HGP_TRY(launch(c, "segsort_cta", k_segsort_cta<Seg>, dim3(2 * c->sm_count), dim3(kCtaSortThreads),
                 kCtaSortCap * 4, seg, (const uint64_t *)big, (const uint32_t *)cnt, keys, huge, cnt + 1));
  if (max_len > kCtaSortCap)
    HGP_TRY(launch(c, "segsort_global", k_segsort_global<Seg>, dim3(c->sm_count), dim3(1024), 0, seg,
                   (const uint64_t *)huge, (const uint32_t *)(cnt + 1), keys));
  return HGP_OK;
}

}  // namespace hgp
