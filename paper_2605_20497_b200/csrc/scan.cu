// scan.cu — second phase of the reduce-then-scan: one CTA scans the tile sums in place.
#include "scan.cuh"

namespace hgp {

__global__ void __launch_bounds__(1024) k_scan_partials(uint64_t *sums, uint32_t nb) {
  __shared__ uint64_t wt[33];
  uint64_t carry = 0;
  for (uint32_t base = 0; base < nb; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint64_t v = i < nb ? sums[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_excl_scan<uint64_t>(v, wt, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}

}  // namespace hgp
