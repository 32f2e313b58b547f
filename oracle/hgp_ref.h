/* hgp_ref — the CPU ORACLE for one coarsening level of arXiv 2605.20497.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2605_20497_b200/, include/hgp.h) never links, imports or calls it, and
 * this oracle shares no code, header, table or helper with the CUDA path.
 *
 * Plain, slow, single-threaded C++17 on HOST arrays (std::vector + std::sort).
 * Every function follows the paper's definition / algorithm in its own order and
 * notation; citations are PAPER.md line numbers (P:n) and SPEC.md lines (S:n).
 * Readings of silent / ambiguous passages are DESIGN.md "Readings" #1-#21.
 *
 * Pinned by tests/test_oracle_*.py against: the SPEC worked examples on H_ex
 * (tests/golden/h_ex.json), brute-force all-pairs scoring via an integer
 * incidence-matrix product, exhaustive matching enumeration, and the
 * coarsening invariants I1-I6 (connectivity / cut-net / Delta-count
 * preservation, duality Score + Conn = sum w(|e|-1)).
 */
#ifndef HGP_REF_H
#define HGP_REF_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define HGP_REF_NONE 0xFFFFFFFFu
#define HGP_REF_UNBOUNDED UINT64_MAX
#define HGP_REF_FP_SHIFT 24
#define HGP_REF_PURGE 0x80000000u

/* status codes (same meanings as the product's, defined independently) */
#define HGP_REF_OK 0
#define HGP_REF_E_ARG (-1)
#define HGP_REF_E_MALFORMED (-2)
#define HGP_REF_E_INFEASIBLE (-3)
#define HGP_REF_E_OVERFLOW (-4)
#define HGP_REF_E_OOM (-5)
#define HGP_REF_E_INTERNAL (-8)

typedef struct {                 /* problem statement, P:290-311 (borrowed host arrays) */
  uint32_t num_nodes, num_edges;
  const uint64_t *edge_off;      /* [E+1] */
  const uint32_t *edge_nsrc;     /* [E]   first nsrc pins of a segment = src(e), rest = dst(e) */
  const uint32_t *pins;          /* [P] */
  const uint32_t *edge_w;        /* [E]   omega(e) >= 1 */
  const uint32_t *node_w;        /* [N]   size(n) >= 1 */
} hgp_ref_input;

typedef struct {                 /* one level, P:479-499 (malloc'd, free with hgp_ref_csr_free) */
  uint32_t N, E;
  uint64_t P;
  uint64_t *edge_off;            /* [E+1] */
  uint32_t *edge_nsrc;           /* [E] */
  uint32_t *pins;                /* [P]  src block ascending, then dst block ascending */
  uint32_t *edge_w;              /* [E]  omega */
  uint32_t *edge_mu;             /* [E]  inbound multiplicity mu (reading #12) */
  uint32_t *node_w;              /* [N]  size */
  uint64_t *inc_off;             /* [N+1] */
  uint32_t *inc_nin;             /* [N]  |in(n)| */
  uint32_t *inc;                 /* [P]  in(n) ascending, then out(n) ascending */
  uint32_t *in_mu;               /* [N]  sum of mu over in(n) */
} hgp_ref_csr;

typedef struct {                 /* materialised neighbours of nodes lo..hi-1 */
  uint32_t lo, hi;
  uint64_t V;
  uint64_t *off;                 /* [hi-lo+1], off[0] = 0 */
  uint32_t *nbr;                 /* [V]  ascending ids, bit31 = purge flag */
} hgp_ref_nbrs;

typedef struct { uint32_t id, pad; uint64_t score; } hgp_ref_cand;   /* [N][pi] */

typedef struct {
  uint64_t omega, delta;         /* Omega, Delta; HGP_REF_UNBOUNDED = +inf */
  uint32_t pi;                   /* Pi candidates per node, 1..16 */
  uint32_t norm;                 /* 0: Eq.5 omega/|e| ; 1: raw omega (reading #1) */
  uint64_t noise_seed, noise_cap;/* noise, cap in 2^-24 units; 0 = off */
  uint32_t batch;                /* neighbour batch size; 0 = whole list */
} hgp_ref_params;

int  hgp_ref_build_csr(const hgp_ref_input *in, hgp_ref_csr *out);
int  hgp_ref_unique_neighbors(const hgp_ref_csr *g, uint32_t lo, uint32_t hi, hgp_ref_nbrs *out);
/* cand: [N*pi]; rows lo..hi-1 written (hi/lo taken from nb). nb flags written in place. */
int  hgp_ref_score_pairs(const hgp_ref_csr *g, hgp_ref_nbrs *nb, const hgp_ref_params *p,
                         hgp_ref_cand *cand);
/* match: [N]; matched_per_round: [pi] pairs matched per round (or NULL);
 * round_value: [pi] DP optimum max(ss-values) summed over components per round (or NULL). */
int  hgp_ref_match(const hgp_ref_cand *cand, uint32_t N, uint32_t pi, uint32_t *match,
                   uint32_t *matched_per_round, int64_t *round_value);
int  hgp_ref_contract(const hgp_ref_csr *g, const hgp_ref_nbrs *nb, const uint32_t *match,
                      uint32_t *gamma, hgp_ref_csr *coarse, hgp_ref_nbrs *coarse_nb);
/* score -> match -> contract on a full-range nb; cand/match/gamma caller-allocated [N*pi]/[N]/[N]. */
int  hgp_ref_coarsen_level(const hgp_ref_csr *g, hgp_ref_nbrs *nb, const hgp_ref_params *p,
                           hgp_ref_cand *cand, uint32_t *match, uint32_t *gamma,
                           hgp_ref_csr *coarse, hgp_ref_nbrs *coarse_nb);
void hgp_ref_csr_free(hgp_ref_csr *g);
void hgp_ref_nbrs_free(hgp_ref_nbrs *nb);
const char *hgp_ref_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
