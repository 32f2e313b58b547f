// scan.cuh — CUB-free device-wide exclusive scan (reduce-then-scan, 3 kernels).
// out[0..n] receives the exclusive prefix sums of f(0..n-1) and out[n] the total.
#pragma once
#include "common.cuh"

namespace hgp {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T *warp_tot, T *total) {
  // returns the exclusive prefix of v over the block; *total = block sum (all threads)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T incl = warp_incl_scan(v);
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    T x = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < (int)(blockDim.x >> 5)) warp_tot[lane] = xi - x;
    if (lane == 31) warp_tot[32] = xi;
  }
  __syncthreads();
  T r = warp_tot[w] + incl - v;
  *total = warp_tot[32];
  __syncthreads();
  return r;
}

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(F f, uint64_t n, uint64_t *block_sums) {
  __shared__ uint64_t wt[33];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += f(base + k);
  uint64_t tot;
  block_excl_scan<uint64_t>(s, wt, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_partials(uint64_t *sums, uint32_t nb);

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_final(F f, uint64_t n, const uint64_t *block_offs,
                                                             uint64_t *out, uint32_t nb) {
  __shared__ uint64_t wt[33];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? f(base + k) : 0;
    s += v[k];
  }
  uint64_t tot;
  uint64_t pre = block_excl_scan<uint64_t>(s, wt, &tot) + block_offs[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = pre;
    pre += v[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = block_offs[nb];
}

// Scan n items of functor f into out[0..n]; returns the total on the host if total != nullptr
// (that read synchronises the stream).
template <class F>
hgp_status scan_exclusive(hgp_ctx *c, F f, uint64_t n, uint64_t *out, uint64_t *total) {
  if (n == 0) {
    HGP_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), c->stream));
    if (total) *total = 0;
    return HGP_OK;
  }
  hgp_status st = HGP_OK;
  const uint32_t nb = div_up(n, kScanTile);
  uint64_t *sums = scratch_raw<uint64_t>(c, (size_t)nb + 1, &st);
  if (!sums) return st;
  HGP_TRY(launch(c, "scan_reduce", k_scan_reduce<F>, dim3(nb), dim3(kScanThreads), 0, f, n, sums));
  HGP_TRY(launch(c, "scan_partials", k_scan_partials, dim3(1), dim3(1024), 0, sums, nb));
  HGP_TRY(launch(c, "scan_final", k_scan_final<F>, dim3(nb), dim3(kScanThreads), 0, f, n,
                 (const uint64_t *)sums, out, nb));
  if (total) HGP_TRY(read_u64(c, out + n, total));
  return HGP_OK;
}

// ---- common scan inputs
struct InU32 {
  const uint32_t *a;
  __device__ uint64_t operator()(uint64_t i) const { return a[i]; }
};
struct InU64 {
  const uint64_t *a;
  __device__ uint64_t operator()(uint64_t i) const { return a[i]; }
};
struct InSum2U32 {   // a[i] + b[i]
  const uint32_t *a, *b;
  __device__ uint64_t operator()(uint64_t i) const { return (uint64_t)a[i] + b[i]; }
};

}  // namespace hgp
