// csr_impl.cuh — helpers shared by the a1 and a5 translation units of the product library.
#pragma once
#include "common.cuh"

namespace hgp {
// Allocate and fill inc_off / inc_nin / inc / in_mu / max_inc of g from its edge arrays.
hgp_status build_incidence(hgp_ctx *c, hgp_csr *g);
// The same by a stable LSD radix sort of (pin << 1 | is_src, edge) pairs (radix.cu); P < 2^30.
hgp_status build_incidence_radix(hgp_ctx *c, hgp_csr *g);
// Stable LSD radix sort of (key, value) u32 pairs by key < 2^kbits (radix.cu); n < 2^30.
hgp_status radix_sort_pairs(hgp_ctx *c, uint32_t *keys, uint32_t *vals, uint32_t *keys_alt, uint32_t *vals_alt,
                            uint64_t n, uint32_t kbits, uint32_t **ko, uint32_t **vo);
// f2 leftover pairing (leftover.cu): extends match in place.
hgp_status leftover_impl(hgp_ctx *c, const hgp_cand *cand, uint32_t N, uint32_t pi, const uint32_t *node_w,
                         const uint32_t *in_mu, uint64_t omega, uint64_t delta, uint32_t *match, uint32_t *added);
void free_csr(hgp_ctx *c, hgp_csr *g);
void free_nbrs(hgp_ctx *c, hgp_nbrs *nb);
// Neighbour segments left in the fused kernel's pool (not compacted into a CSR): segment n is
// nbr[start[n] .. start[n] + len[n]) (scratch of the current top-level call).
struct SegView {
  const uint64_t *start;
  const uint32_t *len;
  const uint32_t *nbr;
  uint64_t V;
};
hgp_status nbrs_for_list(hgp_ctx *c, const hgp_csr *g, uint32_t lo, const uint32_t *list, const uint32_t *list_count,
                         uint32_t hcount, const uint32_t *base, uint64_t *start, uint32_t *cnt, uint32_t *max_deg_out);
hgp_status nbrs_score_fused(hgp_ctx *c, const hgp_csr *g, const hgp_params *p, uint32_t lo, uint32_t hi,
                            hgp_nbrs *out, hgp_cand *cand, SegView *view);
hgp_status contract_impl(hgp_ctx *c, const hgp_csr *g, const hgp_nbrs *nb, const uint32_t *match, uint32_t *gamma,
                         hgp_csr *C, hgp_nbrs *CN, hgp_level_stats *stats, const SegView *view);
}  // namespace hgp
