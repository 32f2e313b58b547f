// pack.cuh — segments (pool + start[t], cnt[t] entries) copied into a CSR (nbr + off[t]) as a flat
// copy balanced by entries: warp w copies the output positions [V w / W, V (w+1) / W), walking the
// segments they span (one binary search over off for the first). A warp per segment left a hub's
// ~10^6 entries to one warp (measured on the coarse-neighbour pack: C4 9.4 -> 2.9 ms).
#pragma once
#include "common.cuh"

namespace hgp {

__global__ void k_seg_pack_flat(const uint32_t *pool, const uint64_t *start, const uint32_t *cnt, const uint64_t *off,
                                uint32_t nn, uint64_t V, uint32_t *nbr, unsigned int *maxdeg);

}  // namespace hgp
