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
/* ---- next rows: f1 partition quality, f3 refinement gains, f4 validation ----
 * part: [N] partition id of every node (rho), every id < nparts. Plain definitions
 * written out; see oracle/hgp_ref_refine.cpp for the passages each follows. */
typedef struct {
  uint64_t connectivity;         /* Eq.1: sum_e omega(e) (lambda(e) - 1) */
  uint64_t cut_net;              /* Eq.16: sum_e omega(e) [lambda(e) > 1] */
  uint64_t max_size;             /* max_p |p| = sum_{n: rho(n)=p} size(n) */
  uint64_t max_inbound;          /* max_p sum_{e: dst(e) meets p} mu(e) (reading #12) */
  uint32_t size_violations;      /* partitions with |p| > Omega */
  uint32_t inbound_violations;   /* partitions with inbound count > Delta */
} hgp_ref_quality;
int hgp_ref_partition_metrics(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, uint64_t omega,
                              uint64_t delta, hgp_ref_quality *out);

/* f3: sparse pins(p, e): per edge e the distinct partitions of its pins in
 * ascending id with their counts; inbound = 1 counts dst(e) pins only (pins_in). */
typedef struct {
  uint32_t E;
  uint64_t nnz;
  uint64_t *off;                 /* [E+1] */
  uint32_t *part;                /* [nnz] ascending inside an edge */
  uint32_t *count;               /* [nnz] >= 1 */
} hgp_ref_pins;
int hgp_ref_pins_matrix(const hgp_ref_csr *g, const uint32_t *part, int inbound, hgp_ref_pins *out);
void hgp_ref_pins_free(hgp_ref_pins *pm);
/* Eq.13 proposals: dest[n] = max_id argmax over p != rho(n) holding a pin of some
 * e in I(n) of gain(n,p) = saving(n) - loss(n,p); HGP_REF_NONE if there is no such p (or none
 * passes size(n) + |p| <= Omega when enforce_size). gain[n] = that gain (0 if none). */
int hgp_ref_propose_moves(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, uint64_t omega,
                          int enforce_size, uint32_t *dest, int64_t *gain);
/* In-sequence gains (Eqs.14-15): seq[0..M) distinct node ids, each with dest[seq[i]]
 * != NONE; gain_seq[i] = connectivity before move i minus after it, with moves 0..i-1 applied. */
int hgp_ref_in_sequence_gains(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, const uint32_t *seq,
                              uint32_t M, const uint32_t *dest, int64_t *gain_seq);
/* f4: violations[i] = number of partitions with |p| > Omega or inbound count > Delta
 * after moves 0..i of the sequence are applied. */
int hgp_ref_sequence_violations(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, const uint32_t *seq,
                                uint32_t M, const uint32_t *dest, uint64_t omega, uint64_t delta,
                                uint32_t *violations);
/* The landing point: *k = the prefix length (1..M) with violations[k-1] == 0 and the
 * largest cumulative in-sequence gain, the shortest on ties; *k = 0 (apply nothing) if that gain is
 * <= 0 or no prefix is legal. *best = its cumulative gain (0 when *k = 0). */
int hgp_ref_best_prefix(const int64_t *gain_seq, const uint32_t *violations, uint32_t M, uint32_t *k, int64_t *best);

void hgp_ref_csr_free(hgp_ref_csr *g);
void hgp_ref_nbrs_free(hgp_ref_nbrs *nb);
const char *hgp_ref_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
