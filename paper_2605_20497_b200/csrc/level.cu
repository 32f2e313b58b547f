// level.cu — hgp_coarsen_level: a3 (score) -> a4 (match) -> a5 (contract) on one level,
// with per-step device times from CUDA events on the ctx stream.
#include "csr_impl.cuh"


using namespace hgp;

extern "C" hgp_status hgp_coarsen_level(hgp_ctx *c, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p, hgp_cand *cand,
                                        uint32_t *match, uint32_t *gamma, hgp_csr *coarse, hgp_nbrs *coarse_nb,
                                        hgp_level_stats *stats) {
  if (!c || !g || !nb || !p || !match || !gamma || !coarse || !coarse_nb)
    return set_error(HGP_E_ARG, "hgp_coarsen_level: null argument");
  if (nb->lo != 0 || nb->hi != g->N) return set_error(HGP_E_ARG, "hgp_coarsen_level: nb must cover every node");
  if (p->pi < 1 || p->pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "pi must be in [1,16]");
  ApiScope scope(c);
  hgp_status st = HGP_OK;
  if (!cand) {
    cand = scratch_raw<hgp_cand>(c, (size_t)g->N * p->pi, &st);
    if (st) return st;
  }
  uint32_t *per = scratch_zero<uint32_t>(c, HGP_MAX_PI, &st);
  if (st) return st;
  HGP_CUDA(cudaEventRecord(c->ev[0], c->stream));
  HGP_TRY(hgp_score_pairs(c, g, nb, p, cand));
  HGP_CUDA(cudaEventRecord(c->ev[1], c->stream));
  HGP_TRY(hgp_match(c, cand, g->N, p->pi, match, per));
  if (p->flags & HGP_FLAG_LEFTOVER)
    HGP_TRY(leftover_impl(c, cand, g->N, p->pi, g->node_w, g->in_mu, p->omega, p->delta, match, nullptr));
  HGP_CUDA(cudaEventRecord(c->ev[2], c->stream));
  hgp_status s = contract_impl(c, g, nb, match, gamma, coarse, coarse_nb, stats, nullptr);
  if (s != HGP_OK) { free_csr(c, coarse); free_nbrs(c, coarse_nb); return s; }
  HGP_CUDA(cudaEventRecord(c->ev[3], c->stream));
  HGP_CUDA(cudaEventSynchronize(c->ev[3]));
  if (stats) {
    stats->N = g->N; stats->E = g->E; stats->P = g->P; stats->V = nb->V;
    uint32_t hper[HGP_MAX_PI];
    HGP_TRY(read_back(c, per, sizeof(hper), hper));
    for (int i = 0; i < HGP_MAX_PI; ++i) stats->matched_per_round[i] = i < (int)p->pi ? hper[i] : 0;
    cudaEventElapsedTime(&stats->ms[0], c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&stats->ms[1], c->ev[1], c->ev[2]);
    cudaEventElapsedTime(&stats->ms[2], c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&stats->ms[3], c->ev[0], c->ev[3]);
  }
  return HGP_OK;
}
