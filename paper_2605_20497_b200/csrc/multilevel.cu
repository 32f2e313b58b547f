// multilevel.cu — hgp_coarsen: the multi-level coarsening driver.
//
// Level 0 runs hgp_coarsen_level0 (fused a2+a3 -> a4 -> a5, N(n) consumed in place); every later
// level runs hgp_coarsen_level on the previous level's coarse CSR and coarse neighbour lists
// (which carry the OR-propagated purge flags, reading #7). Level l uses noise seed
// p->noise_seed + l (reading #3: "the driver passes seed+level"). The driver stops after the
// first level whose coarse node count is <= ceil(W / Omega) (1 when Omega is unbounded), or that
// formed no pair — by a4 or by f2 — i.e. N' = N (reading #20), or after max_levels levels. rho = gamma^L o ... o
// gamma^1 (the initial partition's clusters) is composed on the device.
#include "csr_impl.cuh"

namespace hgp {

__global__ void k_compose(uint32_t *rho, const uint32_t *gamma, uint32_t n0) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n0; i += gridDim.x * blockDim.x) rho[i] = gamma[rho[i]];
}

__global__ void k_iota_u32(uint32_t *a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void k_sum_u32(const uint32_t *a, uint32_t n, unsigned long long *out) {
  uint64_t s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += a[i];
  s = warp_sum(s);
  if (lane_id() == 0 && s) atomicAdd(out, (unsigned long long)s);
}

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_coarsen(hgp_ctx *c, const hgp_csr *g0, const hgp_params *p, uint32_t max_levels,
                                  uint32_t *rho, hgp_csr *coarsest, hgp_nbrs *coarsest_nb, hgp_level_stats *stats,
                                  uint32_t *levels_out) {
  if (!c || !g0 || !p || !rho || !coarsest || !coarsest_nb || !levels_out)
    return set_error(HGP_E_ARG, "hgp_coarsen: null argument");
  DeviceGuard dg(c->device);
  if (max_levels < 1 || max_levels > HGP_MAX_LEVELS) return set_error(HGP_E_ARG, "hgp_coarsen: max_levels must be in [1,64]");
  if (g0->N == 0) return set_error(HGP_E_ARG, "hgp_coarsen: empty hypergraph");
  if (p->pi < 1 || p->pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "pi must be in [1,16]");
  memset(coarsest, 0, sizeof(*coarsest));
  memset(coarsest_nb, 0, sizeof(*coarsest_nb));
  *levels_out = 0;
  const uint32_t N0 = g0->N;
  const uint32_t grid = div_up(N0, 256) < 4096 ? div_up(N0, 256) : 4096;
  // stop rule (reading #20): ceil(W / Omega) coarse nodes, W = total size
  uint64_t stop = 1;
  {
    hgp_status st = HGP_OK;
    unsigned long long *d = nullptr;
    {
      ApiScope scope(c);
      d = scratch_zero<unsigned long long>(c, 1, &st);
      if (st) return st;
      HGP_TRY(launch(c, "sum_w", k_sum_u32, dim3(grid), dim3(256), 0, (const uint32_t *)g0->node_w, N0, d));
      uint64_t W = 0;
      HGP_TRY(read_u64(c, (const uint64_t *)d, &W));
      if (p->omega != HGP_UNBOUNDED) stop = p->omega ? (W + p->omega - 1) / p->omega : W;
      if (stop < 1) stop = 1;
    }
  }
  HGP_TRY(launch(c, "iota", k_iota_u32, dim3(grid), dim3(256), 0, rho, N0));
  // per-level device buffers (match, gamma at the level's N <= N0)
  hgp_status st = HGP_OK;
  uint32_t *match = dalloc_n<uint32_t>(c, N0, &st);
  uint32_t *gamma = dalloc_n<uint32_t>(c, N0, &st);
  if (st) { if (match) c->dfree(match, 4ull * N0); if (gamma) c->dfree(gamma, 4ull * N0); return st; }
  auto release = [&]() { c->dfree(match, 4ull * N0); c->dfree(gamma, 4ull * N0); };
  hgp_csr cur{};
  hgp_nbrs cur_nb{};
  bool own = false;                                  // cur is library-owned (level >= 1)
  hgp_status s = HGP_OK;
  for (uint32_t lvl = 0; lvl < max_levels; ++lvl) {
    hgp_params pl = *p;
    pl.noise_seed = p->noise_seed + lvl;
    hgp_csr nxt{};
    hgp_nbrs nxt_nb{};
    hgp_level_stats ls{};
    if (lvl == 0) s = hgp_coarsen_level0(c, g0, &pl, nullptr, match, gamma, nullptr, &nxt, &nxt_nb, &ls);
    else s = hgp_coarsen_level(c, &cur, &cur_nb, &pl, nullptr, match, gamma, &nxt, &nxt_nb, &ls);
    if (s != HGP_OK) break;
    const uint32_t nl = lvl == 0 ? N0 : cur.N;
    {
      ApiScope scope(c);
      s = launch(c, "compose", k_compose, dim3(grid), dim3(256), 0, rho, (const uint32_t *)gamma, N0);
    }
    if (own) { free_csr(c, &cur); free_nbrs(c, &cur_nb); }
    cur = nxt;
    cur_nb = nxt_nb;
    own = true;
    if (stats) stats[lvl] = ls;
    *levels_out = lvl + 1;
    if (s != HGP_OK) break;
    // no pair formed on this level (a4 rounds and, with HGP_FLAG_LEFTOVER, f2 pairs alike): N' = N
    if ((uint64_t)cur.N <= stop || cur.N == nl) break;
  }
  release();
  if (s != HGP_OK) {
    if (own) { free_csr(c, &cur); free_nbrs(c, &cur_nb); }
    return s;
  }
  *coarsest = cur;
  *coarsest_nb = cur_nb;
  return hgp_sync(c);
}
