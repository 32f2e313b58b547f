// leftover.cu — f2: deterministic best-effort pairing of the nodes left without any candidate
// (DESIGN reading #22).
//
// "After the above proposal completes, all such nodes are gathered and sorted by size. Each node
// ... runs a binary search for its current cluster size slack and tries to ... claim the first
// valid node it finds. Contentions are broken by id. ... inbound set union sizes are
// overestimated with the sum of each node's inbound set size." The atomic claims are replaced by
// the exact a4 DP: every leftover n targets the valid leftover m with the largest (size, id)
// (binary search on the size-sorted list, then a downward walk to the first node passing the
// inbound over-estimate), score size(n) + size(m); the symmetric score with consistent ties makes
// the proposal graph a two-cycle pseudo-forest, solved by hgp_match as one round (pi = 1).
#include "csr_impl.cuh"
#include "scan.cuh"

namespace hgp {

__global__ void k_left_flags(const hgp_cand *cand, uint32_t N, uint32_t pi, uint32_t *flag) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    flag[n] = cand[(uint64_t)n * pi].id == kNone ? 1u : 0u;
}

// L in ascending id order (scan positions), keyed by size for the stable sort
__global__ void k_left_gather(const uint32_t *flag, const uint64_t *pos, uint32_t N, const uint32_t *node_w,
                              uint32_t *keys, uint32_t *vals) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    if (flag[n]) { keys[pos[n]] = node_w[n]; vals[pos[n]] = n; }
}

__global__ void k_left_none(hgp_cand *c2, uint32_t N) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    hgp_cand cd;
    cd.id = kNone; cd.pad = 0; cd.score = 0;
    c2[n] = cd;
  }
}

// One thread per leftover (sorted position i): the largest (size, id) valid partner.
__global__ void k_left_target(const uint32_t *skeys, const uint32_t *svals, uint32_t L, const uint32_t *in_mu,
                              uint64_t omega, uint64_t delta, hgp_cand *c2) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const uint32_t n = svals[i];
    const uint64_t wn = skeys[i];
    if (wn > omega) continue;
    const uint64_t slack = omega - wn;
    // last position j with size <= slack (sizes ascending)
    uint32_t lo = 0, hi = L;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((uint64_t)skeys[mid] <= slack) lo = mid + 1; else hi = mid;
    }
    const uint64_t inn = in_mu[n];
    for (int64_t j = (int64_t)lo - 1; j >= 0; --j) {
      if ((uint32_t)j == i) continue;
      const uint32_t m = svals[j];
      if (delta != HGP_UNBOUNDED && inn + in_mu[m] > delta) continue;   // inbound over-estimate
      hgp_cand cd;
      cd.id = m; cd.pad = 0; cd.score = wn + skeys[j];
      c2[n] = cd;
      break;
    }
  }
}

__global__ void k_left_merge(const uint32_t *m2, uint32_t N, uint32_t *match) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    if (m2[n] != kNone) match[n] = m2[n];
}

hgp_status leftover_impl(hgp_ctx *c, const hgp_cand *cand, uint32_t N, uint32_t pi, const uint32_t *node_w,
                         const uint32_t *in_mu, uint64_t omega, uint64_t delta, uint32_t *match, uint32_t *added) {
  if (N == 0) return HGP_OK;
  hgp_status st = HGP_OK;
  const uint32_t grid = div_up(N, 256) < 4096 ? div_up(N, 256) : 4096;
  uint32_t *flag = scratch_raw<uint32_t>(c, N, &st);
  uint64_t *pos = scratch_raw<uint64_t>(c, (size_t)N + 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "left_flags", k_left_flags, dim3(grid), dim3(256), 0, cand, N, pi, flag));
  uint64_t L = 0;
  HGP_TRY(scan_exclusive(c, InU32{flag}, N, pos, &L));
  hgp_cand *c2 = scratch_raw<hgp_cand>(c, N, &st);
  uint32_t *m2 = scratch_raw<uint32_t>(c, N, &st);
  uint32_t *per = scratch_zero<uint32_t>(c, 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "left_none", k_left_none, dim3(grid), dim3(256), 0, c2, N));
  if (L >= 2) {
    uint32_t *k0 = scratch_raw<uint32_t>(c, L, &st), *v0 = scratch_raw<uint32_t>(c, L, &st);
    uint32_t *k1 = scratch_raw<uint32_t>(c, L, &st), *v1 = scratch_raw<uint32_t>(c, L, &st);
    if (st) return st;
    HGP_TRY(launch(c, "left_gather", k_left_gather, dim3(grid), dim3(256), 0, (const uint32_t *)flag,
                   (const uint64_t *)pos, N, node_w, k0, v0));
    uint32_t *ks = nullptr, *vs = nullptr;
    HGP_TRY(radix_sort_pairs(c, k0, v0, k1, v1, L, 32, &ks, &vs));   // stable: (size, id) ascending
    const uint32_t gl = div_up(L, 128) < 4096 ? div_up(L, 128) : 4096;
    HGP_TRY(launch(c, "left_target", k_left_target, dim3(gl), dim3(128), 0, (const uint32_t *)ks,
                   (const uint32_t *)vs, (uint32_t)L, in_mu, omega, delta, c2));
  }
  HGP_TRY(hgp_match(c, c2, N, 1, m2, per));
  HGP_TRY(launch(c, "left_merge", k_left_merge, dim3(grid), dim3(256), 0, (const uint32_t *)m2, N, match));
  if (added) HGP_CUDA(cudaMemcpyAsync(added, per, 4, cudaMemcpyDeviceToDevice, c->stream));
  return HGP_OK;
}

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_leftover_pairs(hgp_ctx *c, const hgp_cand *cand, uint32_t N, uint32_t pi,
                                         const uint32_t *node_w, const uint32_t *in_mu, uint64_t omega,
                                         uint64_t delta, uint32_t *match, uint32_t *added) {
  if (!c || (N && (!cand || !node_w || !in_mu || !match))) return set_error(HGP_E_ARG, "hgp_leftover_pairs: null argument");
  if (pi < 1 || pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "pi must be in [1,16]");
  ApiScope scope(c);
  return leftover_impl(c, cand, N, pi, node_w, in_mu, omega, delta, match, added);
}
