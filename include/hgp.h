/* hgp.h — C-ABI of the B200-native coarsening level (arXiv 2605.20497, §5).
 *
 * One coarsening level of a weighted directed hypergraph under a size limit Omega
 * and a distinct-inbound-hyperedge limit Delta, as five steps:
 *   a1 hgp_build_csr        compressed sparse layout, src-first / in-first
 *   a2 hgp_unique_neighbors materialised unique neighbourhoods N(n)
 *   a3 hgp_score_pairs      histogram eta + inline intersection + validity + noise
 *                           + purge flags + top-Pi candidates (Eqs.5-6)
 *   a4 hgp_match            exact DP matching on Pi two-cycle pseudo-forests (Eqs.7-12)
 *   a5 hgp_contract         gamma + coarse hyperedges/incidence/neighbours
 * and hgp_coarsen_level = a3 -> a4 -> a5 on one level.
 *
 * Conventions
 *  - Every pointer inside hgp_input / hgp_csr / hgp_nbrs / hgp_cand / match / gamma is a
 *    DEVICE pointer on the ctx's device. Host pointers appear only where stated.
 *  - Ids are uint32; HGP_NONE marks "undefined". Node count N < 2^31 (bit 31 of a
 *    neighbour entry is the purge flag).
 *  - Scores are unsigned fixed point with HGP_FP_SHIFT fraction bits: the Eq.5 term of
 *    an edge is c(e) = floor(omega(e) * 2^24 / |e|) (norm = 0) or omega(e) * 2^24 (norm = 1).
 *    All sums are exact integers, so results do not depend on the parallel schedule.
 *  - Ownership: inputs are borrowed (they must stay alive until the stream passes the
 *    call); fixed-size outputs (cand, match, gamma) are caller-allocated; data-dependent
 *    outputs (hgp_csr, hgp_nbrs arrays) are allocated by the library through the ctx's
 *    allocator and released with hgp_csr_free / hgp_nbrs_free.
 *  - Order inside a segment: hyperedge src/dst blocks and incidence in/out lists are
 *    ascending (canonical). Neighbour segments are SETS (ascending order is not
 *    guaranteed; the paper builds them with hash sets); compare them as sets.
 *  - Errors: every call returns an hgp_status; the first error wins and
 *    hgp_last_error() (thread-local) names the lowest offending edge/node index.
 *    No exceptions and no host fallback: without a CUDA device every call fails.
 *  - Synchronisation: EVERY compute entry point synchronises the ctx stream before it
 *    returns, because each one reads device values on the host: hgp_build_csr,
 *    hgp_unique_neighbors, hgp_contract (scan totals size their outputs), hgp_score_pairs
 *    (work totals pick the kernel tier; the infeasibility check of P:321 is returned as a
 *    status), hgp_match (the per-round count of over-long best-child chains selects the
 *    pointer-jumping fallback; the two-cycle check of P:546-547 is returned as a status).
 *    Outputs are therefore complete and errors final when a call returns; callers overlap
 *    work across ctxs on different streams, not within one call.
 *  - Device: every call makes the ctx's device current for its duration and restores the
 *    caller's current device before returning (hgp_ctx_create included).
 */
#ifndef HGP_H
#define HGP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define HGP_API
#else
#define HGP_API __attribute__((visibility("default")))
#endif

#define HGP_NONE 0xFFFFFFFFu
#define HGP_UNBOUNDED UINT64_MAX          /* Omega or Delta = +inf (k-way: Delta) */
#define HGP_FP_SHIFT 24
#define HGP_PURGE 0x80000000u             /* neighbour entry flag: permanently invalid */
#define HGP_MAX_PI 16
#define HGP_MAX_LEVELS 64   /* hgp_coarsen: at most this many levels */
#define HGP_FLAG_LEFTOVER 1u /* hgp_params.flags: run hgp_leftover_pairs after a4 */

typedef enum {
  HGP_OK = 0,
  HGP_E_ARG = -1,         /* bad argument (null pointer, range, parameter out of domain) */
  HGP_E_MALFORMED = -2,   /* input violates P:290-297: pin >= N, duplicate pin, src∩dst != ∅,
                             empty edge, omega = 0, size = 0, non-monotone offsets, nsrc > |e| */
  HGP_E_INFEASIBLE = -3,  /* a node alone exceeds Omega or Delta: no valid solution */
  HGP_E_OVERFLOW = -4,    /* N >= 2^31, |e| > 2^24, sum omega >= 2^32, sum size >= 2^32,
                             or score totals that could reach 2^62 */
  HGP_E_OOM = -5,         /* the allocator returned NULL */
  HGP_E_CUDA = -6,        /* CUDA runtime error (message carries cudaGetErrorString) */
  HGP_E_NCCL = -7,        /* reserved for the library-internal NCCL path */
  HGP_E_INTERNAL = -8     /* broken invariant, e.g. a proposal cycle longer than 2 */
} hgp_status;

typedef struct CUstream_st *hgp_stream_t;   /* == cudaStream_t */

/* Device allocator. alloc returns a device pointer (NULL on failure); free releases it.
 * Both are called on the host thread that issued the hgp_* call, with the ctx stream.
 * Passing NULL to hgp_ctx_create selects the built-in stream-ordered pool (cudaMallocAsync). */
typedef struct {
  void *(*alloc)(void *user, size_t bytes, hgp_stream_t stream);
  void (*free)(void *user, void *ptr, size_t bytes, hgp_stream_t stream);
  void *user;
} hgp_allocator;

typedef struct hgp_ctx hgp_ctx;             /* opaque: device, stream, allocator, scratch arena */

/* Problem statement. DEVICE pointers, borrowed. */
typedef struct {
  uint32_t num_nodes, num_edges;
  const uint64_t *edge_off;   /* [E+1] edge_off[0] = 0, nondecreasing; |e| = off[e+1]-off[e] >= 1 */
  const uint32_t *edge_nsrc;  /* [E]   the first nsrc pins of edge e are src(e), the rest dst(e) */
  const uint32_t *pins;       /* [P]   node ids < N, any order inside the src / dst blocks */
  const uint32_t *edge_w;     /* [E]   omega(e) >= 1, sum < 2^32 */
  const uint32_t *node_w;     /* [N]   size(n) >= 1, sum < 2^32 */
} hgp_input;

/* One level. Library-owned DEVICE arrays; scalar fields are host values. */
typedef struct {
  uint32_t N, E;
  uint64_t P;                 /* number of pins = sum |e| = sum |I(n)| */
  uint32_t max_edge;          /* max |e| (host-known, selects kernel tiers) */
  uint32_t max_inc;           /* max |I(n)| */
  uint64_t *edge_off;         /* [E+1] */
  uint32_t *edge_nsrc;        /* [E]   |src(e)| */
  uint32_t *pins;             /* [P]   src(e) ascending ‖ dst(e) ascending */
  uint32_t *edge_w;           /* [E]   omega(e) (coarse: sum over merged edges) */
  uint32_t *edge_mu;          /* [E]   inbound multiplicity: original edges merged into e */
  uint32_t *node_w;           /* [N]   size(n) */
  uint64_t *inc_off;          /* [N+1] */
  uint32_t *inc_nin;          /* [N]   |in(n)| */
  uint32_t *inc;              /* [P]   in(n) ascending ‖ out(n) ascending (edge ids) */
  uint32_t *in_mu;            /* [N]   sum of mu(e) over in(n) = distinct original inbound edges */
} hgp_csr;

/* Materialised neighbours of nodes lo..hi-1. Library-owned DEVICE arrays. */
typedef struct {
  uint32_t lo, hi;
  uint64_t V;                 /* entries */
  uint32_t max_deg;           /* max |N(n)| over the range (host-known) */
  uint32_t pad_;
  uint64_t *off;              /* [hi-lo+1], off[0] = 0 */
  uint32_t *nbr;              /* [V]   node id | HGP_PURGE flag; each segment is a set */
} hgp_nbrs;

/* Candidate: node-major [N][pi]; unused slots id = HGP_NONE, score = 0. */
typedef struct { uint32_t id, pad; uint64_t score; } hgp_cand;

typedef struct {
  uint64_t omega, delta;      /* Omega, Delta (HGP_UNBOUNDED allowed); validity uses <= */
  uint32_t pi;                /* Pi in [1, 16]; the paper's default is 4 */
  uint32_t norm;              /* 0: Eq.5 omega/|e| (default); 1: raw omega */
  uint64_t noise_seed;        /* deterministic symmetric noise */
  uint64_t noise_cap;         /* noise in [0, cap], 2^-24 units; 0 disables; cap < 2^56 */
  uint32_t batch;             /* tuning only; results never depend on it */
  uint32_t flags;             /* HGP_FLAG_* bits; 0 = the level exactly as §8(a) defines it */
} hgp_params;

typedef struct {
  uint32_t N, E, Nc, Ec;
  uint64_t P, V, Pc, Vc;
  uint32_t matched_per_round[HGP_MAX_PI];
  uint32_t dropped_edges, merged_edges;
  uint64_t purged;            /* entries flagged by a3 in this level */
  float ms[4];                /* device time: score, match, contract, total (CUDA events) */
} hgp_level_stats;

/* ---- context ---------------------------------------------------------------------------- */
/* device: CUDA ordinal; stream: NULL = the legacy default stream; alloc: NULL = built-in pool. */
HGP_API hgp_status hgp_ctx_create(int device, hgp_stream_t stream, const hgp_allocator *alloc, hgp_ctx **out);
HGP_API void hgp_ctx_destroy(hgp_ctx *ctx);
HGP_API const char *hgp_last_error(void);
/* number of kernels this ctx has launched so far (for the bench's gpu_launches claim) */
HGP_API uint64_t hgp_launch_count(const hgp_ctx *ctx);
/* stream-ordered copy on the ctx stream, cudaMemcpyDefault semantics (host or device pointers);
 * synchronises the stream when either side is pageable host memory. */
HGP_API hgp_status hgp_copy(hgp_ctx *ctx, void *dst, const void *src, size_t bytes);
HGP_API hgp_status hgp_sync(hgp_ctx *ctx);
/* Explicit per-ctx options (tests and experiments; the library reads no environment variables).
 * Results never depend on them. Names: "fused_sample_min" (level size from which the fused
 * level-0 kernel first runs tier A on every 64th node; default 65536), "fused_pool_cap" (capacity of
 * the fused kernel's first neighbour pool, 0 = automatic), "unfused" (1: every node takes the
 * unfused a2 -> a3 path), "inc_radix" (1: incidence transpose by radix sort), "debug_sync" (1:
 * synchronise and trace every launch on stderr), "no_hub" (1: hub nodes on the global-memory tiers
 * instead of the key-partitioned hub tiers). Unknown names and negative values: HGP_E_ARG. */
HGP_API hgp_status hgp_ctx_set_option(hgp_ctx *ctx, const char *name, int64_t value);
/* Instrumentation: from hgp_profile_begin on, every kernel launch whose internal name contains
 * name_filter (e.g. "score_A") is bracketed by CUDA events on the ctx stream; hgp_profile_end
 * synchronises and returns the summed device time (ms) and the number of such launches. */
HGP_API hgp_status hgp_profile_begin(hgp_ctx *ctx, const char *name_filter);
HGP_API hgp_status hgp_profile_end(hgp_ctx *ctx, double *total_ms, uint64_t *launches);
/* After hgp_profile_end: per kernel name "name:ms:launches;" into the HOST buffer buf. */
HGP_API hgp_status hgp_profile_report(hgp_ctx *ctx, char *buf, size_t len);

/* Work counters per kernel tier (tests: every tier is exercised). Counter i counts the
 * nodes (or node rounds) the tier processed since the ctx was created or last reset; the
 * counting costs one atomic per CTA per launch. Indices: */
enum {
  HGP_TIER_FUSED_S = 0,      /* fused a2+a3, sampled first tier (every 64th node) */
  HGP_TIER_FUSED_A = 1,      /* fused a2+a3, 4096-slot table */
  HGP_TIER_FUSED_M = 2,      /* fused a2+a3, 8192-slot table */
  HGP_TIER_FUSED_B = 3,      /* fused a2+a3, 16384-slot table */
  HGP_TIER_NBRS_1 = 4,       /* a2 unfused, smem tier 1 (range and list forms) */
  HGP_TIER_NBRS_2 = 5,       /* a2 unfused, smem tier 2 */
  HGP_TIER_NBRS_3 = 6,       /* a2 unfused, global-memory tables */
  HGP_TIER_SCORE_NOINTER = 7, /* a3 first tier, eta only (Delta test cannot fail) */
  HGP_TIER_SCORE_PACKED = 8, /* a3 first tier, (eta/g) << ib | inter in one u32 */
  HGP_TIER_SCORE_SPLIT = 9,  /* a3 first tier, u32 eta + u16 inter */
  HGP_TIER_SCORE_B = 10,     /* a3 big neighbourhoods, packed */
  HGP_TIER_SCORE_W = 11,     /* a3 64-bit eta, smem */
  HGP_TIER_SCORE_H = 12,     /* a3 64-bit eta, global-memory tables */
  HGP_TIER_CNBRS_A = 13,     /* a5 coarse neighbours, 4096-slot table */
  HGP_TIER_CNBRS_M = 14,     /* a5 coarse neighbours, 16384-slot table */
  HGP_TIER_CNBRS_B = 15,     /* a5 coarse neighbours, 32768-slot table */
  HGP_TIER_CNBRS_C = 16,     /* a5 coarse neighbours, global-memory tables */
  HGP_TIER_JUMP = 17,        /* a4 pointer-jumping fallback (nodes of over-long best-child chains) */
  HGP_TIER_FUSED_W = 18,     /* fused a2+a3, one warp per small node (<= 256 pin visits) */
  HGP_TIER_FUSED_H = 19,     /* fused a2+a3, hub nodes: key-partitioned shared tables (hub.cu) */
  HGP_TIER_CNBRS_H = 20,     /* a5 coarse neighbours of hub coarse nodes, key-partitioned */
  HGP_TIER_CNBRS_A2 = 21,    /* a5 coarse neighbours, 8192-slot table (between A and M) */
  HGP_TIER_SCORE_HUB = 22,   /* a3 on big N(n) (> 2048), key-partitioned shared tables (score_hub.cu) */
  HGP_TIERS = 24
};
/* HOST out[HGP_TIERS] <- the counters (synchronises); reset != 0 zeroes them afterwards. */
HGP_API hgp_status hgp_tier_counts(hgp_ctx *ctx, uint64_t *out, int reset);

/* ---- the level's steps ------------------------------------------------------------------ */
/* a1: validate the input and build the canonical level-0 CSR (mu = 1). Synchronises. */
HGP_API hgp_status hgp_build_csr(hgp_ctx *ctx, const hgp_input *in, hgp_csr *out);

/* a2: N(n) = (U_{e in I(n)} e) \ {n} for n in [lo, hi), purge bits clear. Synchronises. */
HGP_API hgp_status hgp_unique_neighbors(hgp_ctx *ctx, const hgp_csr *g, uint32_t lo, uint32_t hi,
                                        hgp_nbrs *out);

/* a3: for n in [nb->lo, nb->hi): eta/inter histogram over unflagged N(n), validity, noise,
 * purge flags set IN PLACE on nb (idempotent), top-pi valid neighbours by (score desc, id desc)
 * into cand rows lo..hi-1 of a caller [N][pi] array. Synchronises; HGP_E_INFEASIBLE names the
 * lowest node that alone exceeds Omega or Delta. */
HGP_API hgp_status hgp_score_pairs(hgp_ctx *ctx, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p,
                                   hgp_cand *cand);

/* a4: pi rounds of exact matching; match[N] symmetric partner or HGP_NONE;
 * matched_per_round: DEVICE [pi] pairs matched per round, or NULL. Synchronises;
 * HGP_E_INTERNAL names a node on a proposal cycle longer than 2 (cannot happen for cand from a3). */
HGP_API hgp_status hgp_match(hgp_ctx *ctx, const hgp_cand *cand, uint32_t N, uint32_t pi,
                             uint32_t *match, uint32_t *matched_per_round);

/* a5: gamma[N] (coarse ids by ascending min member) and the coarse level: merged parallel
 * edges (omega' = sum omega, mu' = sum mu, ordered by min fine edge id), canonical incidence,
 * coarse neighbours = gamma(N(a) ∪ N(b)) minus OR-propagated purged entries minus self.
 * nb must cover every node. Synchronises. */
HGP_API hgp_status hgp_contract(hgp_ctx *ctx, const hgp_csr *g, const hgp_nbrs *nb, const uint32_t *match,
                                uint32_t *gamma, hgp_csr *coarse, hgp_nbrs *coarse_nb);

/* a3 -> a4 -> a5 on one level. cand may be NULL (scratch). stats (HOST pointer) may be NULL. */
HGP_API hgp_status hgp_coarsen_level(hgp_ctx *ctx, const hgp_csr *g, hgp_nbrs *nb, const hgp_params *p,
                                     hgp_cand *cand, uint32_t *match, uint32_t *gamma, hgp_csr *coarse,
                                     hgp_nbrs *coarse_nb, hgp_level_stats *stats);

/* a2 + a3 fused for nodes [lo, hi) of a level whose neighbour lists carry no flags yet (the
 * first level): one traversal of I(n) builds N(n) and its histogram together (level0.cu).
 * Outputs are identical to hgp_unique_neighbors(g, lo, hi) followed by hgp_score_pairs; nodes
 * the fused kernel cannot represent make the call run that unfused pair instead. nb (covering
 * lo..hi) is allocated by the library; cand is caller [N][pi], rows lo..hi-1 written.
 * Synchronises. */
HGP_API hgp_status hgp_neighbors_and_scores(hgp_ctx *ctx, const hgp_csr *g, const hgp_params *p, uint32_t lo,
                                           uint32_t hi, hgp_nbrs *nb, hgp_cand *cand);

/* Node-range sharding for multi-GPU (north_star: "scoring and matching shard by node range over
 * a replicated CSR"): bounds[0..world] (HOST) splits [0, N) into contiguous ranges of about equal
 * traversal work sum_{e in I(n)} |e|. Deterministic (depends on the replicated CSR only). */
HGP_API hgp_status hgp_shard_bounds(hgp_ctx *ctx, const hgp_csr *g, uint32_t world, uint32_t *bounds);

/* The first level straight from a level-0 CSR: fused a2+a3 -> a4 -> a5. nb receives N(n) with
 * the purge flags set by a3 (library-owned); nb may be NULL, in which case N(n) is consumed by a5
 * where the fused kernel left it (no compaction pass) and not returned. cand may be NULL;
 * stats (HOST) may be NULL. */
HGP_API hgp_status hgp_coarsen_level0(hgp_ctx *ctx, const hgp_csr *g, const hgp_params *p, hgp_cand *cand,
                                      uint32_t *match, uint32_t *gamma, hgp_nbrs *nb, hgp_csr *coarse,
                                      hgp_nbrs *coarse_nb, hgp_level_stats *stats);

/* f2 (DESIGN reading #22): deterministic best-effort pairing of the
 * nodes left without any candidate (cand[n][0].id == HGP_NONE; a4 never matches them). Each such n
 * targets the other such m with the largest (node_w[m], m) satisfying node_w[n] + node_w[m] <= omega
 * and in_mu[n] + in_mu[m] <= delta (the paper's over-estimate of the inbound union); score
 * node_w[n] + node_w[m]; the resulting two-cycle pseudo-forest is solved by the a4 DP as one round
 * and merged into match (DEVICE [N], in/out). cand: DEVICE [N][pi] from a3; node_w, in_mu: DEVICE
 * [N] of the level; added: DEVICE [1] pairs added, or NULL. Synchronises (scan totals). */
HGP_API hgp_status hgp_leftover_pairs(hgp_ctx *ctx, const hgp_cand *cand, uint32_t N, uint32_t pi,
                                      const uint32_t *node_w, const uint32_t *in_mu, uint64_t omega,
                                      uint64_t delta, uint32_t *match, uint32_t *added);

/* Multi-level coarsening driver (paper §5): level 0 by
 * hgp_coarsen_level0, level l >= 1 by hgp_coarsen_level on the previous coarse CSR and coarse
 * neighbour lists, noise seed p->noise_seed + l (reading #3). Stops after the first level whose
 * coarse node count is <= ceil(W / Omega) (1 if Omega = HGP_UNBOUNDED; W = total size) or that
 * formed no pair, by a4 or by f2 (N' = N; reading #20), or after max_levels (1..HGP_MAX_LEVELS) levels.
 *   rho        caller DEVICE [g0->N]: rho = gamma^L o ... o gamma^1, each level-0 node's node on
 *              the coarsest level (the initial partition's clusters)
 *   coarsest, coarsest_nb   library-owned coarsest level (free with hgp_csr_free / hgp_nbrs_free)
 *   stats      HOST [max_levels] per-level stats, or NULL; *levels_out = L (number of levels run)
 * g0 is borrowed and left unchanged. Errors of a level are returned as is (nothing is
 * allocated on error). Synchronises. */
HGP_API hgp_status hgp_coarsen(hgp_ctx *ctx, const hgp_csr *g0, const hgp_params *p, uint32_t max_levels,
                               uint32_t *rho, hgp_csr *coarsest, hgp_nbrs *coarsest_nb, hgp_level_stats *stats,
                               uint32_t *levels_out);

/* ---- a5 in pieces, for node/edge-range shards over several GPUs --------------
 * hgp_contract is hgp_gamma + hgp_contract_edges(all edges) + hgp_contract_merge +
 * hgp_coarse_neighbors(all coarse nodes) on one GPU. On W GPUs every rank holds the replicated
 * fine CSR and match (a4 is replicated), builds the coarse edges of its fine edge range, the
 * ranges' hgp_cedges are all-gathered in rank order (= ascending fine edge id; the caller's
 * collective, e.g. NCCL through torch.distributed), the merge runs replicated, and each rank builds
 * the coarse neighbours of the coarse nodes whose min member it owns — the partner's N(b) comes
 * from its owner by a halo exchange (the caller's point-to-point). Results equal hgp_contract's. */

/* gamma (reading #11) of a symmetric match: DEVICE gamma[N]; *Nc (HOST) = N'. */
HGP_API hgp_status hgp_gamma(hgp_ctx *ctx, const uint32_t *match, uint32_t N, uint32_t *gamma, uint32_t *Nc);

/* Coarse node ranges of node-range shards: coarse_bounds[i] (HOST) = number of coarse nodes whose
 * min member is < node_bounds[i] (HOST [nbounds], each <= N): the coarse nodes a rank owning
 * [b_r, b_{r+1}) builds the neighbours of are [coarse_bounds[r], coarse_bounds[r+1]). */
HGP_API hgp_status hgp_coarse_bounds(hgp_ctx *ctx, const uint32_t *match, uint32_t N, const uint32_t *node_bounds,
                                     uint32_t nbounds, uint32_t *coarse_bounds);

/* Coarse edges of the fine edges [elo, ehi) before the parallel-edge merge: for every
 * kept fine edge (D' != ∅ or |S'| >= 2, reading #14), ascending. Library-owned DEVICE arrays. */
typedef struct {
  uint32_t K, pad_;            /* kept fine edges */
  uint64_t P;                  /* sum of their coarse sizes */
  uint32_t *eid;               /* [K]   fine edge id, ascending */
  uint64_t *fp;                /* [K]   64-bit fingerprint of (|S'|, S', D') (hash only; equality is verified) */
  uint32_t *nsrc;              /* [K]   |S'| */
  uint32_t *size;              /* [K]   |S'| + |D'| */
  uint64_t *off;               /* [K+1] */
  uint32_t *pins;              /* [P]   S' ascending ‖ D' ascending, per edge */
} hgp_cedges;
HGP_API hgp_status hgp_contract_edges(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *gamma, uint32_t elo,
                                      uint32_t ehi, hgp_cedges *out);
HGP_API void hgp_cedges_free(hgp_ctx *ctx, hgp_cedges *ce);

/* The coarse level's edges and incidence from `all` (every range's hgp_cedges concatenated in
 * ascending fine id, offsets rebased; DEVICE arrays borrowed): identical (S', D') merged (omega' and
 * mu' summed, ordered by the minimum fine id; reading #12); gamma (DEVICE [N]) recomputed from match;
 * coarse node sizes. coarse is library-owned (hgp_csr_free). */
HGP_API hgp_status hgp_contract_merge(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *match, uint32_t *gamma,
                                      const hgp_cedges *all, hgp_csr *coarse);

/* Coarse neighbours (readings #7, #16) of the coarse nodes [clo, chi): for c with
 * members a (min) and b, gamma(N(a) ∪ N(b)) minus OR-flagged entries minus c. Fine node n's N(n)
 * is nbr[seg_start[n] .. seg_start[n] + seg_len[n]) (DEVICE [N] arrays; only members of
 * [clo, chi) are read). out covers [clo, chi) (library-owned). */
HGP_API hgp_status hgp_coarse_neighbors(hgp_ctx *ctx, const uint32_t *match, const uint32_t *gamma, uint32_t N,
                                        const uint64_t *seg_start, const uint32_t *seg_len, const uint32_t *nbr,
                                        uint32_t clo, uint32_t chi, hgp_nbrs *out);

/* ---- rows after the level: f1 quality, f3 refinement gains, f4 validation ----
 * A partition is part[N] (DEVICE) with ids < nparts; any id >= nparts is HGP_E_ARG naming the
 * lowest such node. Every call synchronises. All sums are exact integers. */

/* f1: quality of a partition (HOST struct). */
typedef struct {
  uint64_t connectivity;        /* Eq.1: sum over e of omega(e) (lambda(e) - 1) */
  uint64_t cut_net;             /* Eq.16: sum of omega(e) over edges with lambda(e) > 1 */
  uint64_t max_size;            /* max over p of sum of size(n), n in p */
  uint64_t max_inbound;         /* max over p of sum of mu(e) over e with a dst pin in p */
  uint32_t size_violations;     /* partitions with size > Omega */
  uint32_t inbound_violations;  /* partitions with inbound load > Delta (never for HGP_UNBOUNDED) */
} hgp_quality;

/* f3: sparse pins(p, e) or pins_in(p, e): row e lists the distinct partitions
 * of e's pins (of dst(e) only for pins_in) in ascending id with their pin counts. Library-owned
 * DEVICE arrays, released with hgp_pins_free. lambda(e) = off[e+1] - off[e] for the full matrix. */
typedef struct {
  uint32_t E, pad_;
  uint64_t nnz;
  uint64_t *off;                /* [E+1] */
  uint32_t *part;               /* [nnz] */
  uint32_t *count;              /* [nnz] >= 1 */
} hgp_pins;

/* f3: the pins matrix of part on level g (inbound = 0: all pins; 1: dst pins only). */
HGP_API hgp_status hgp_pins_matrix(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                   int inbound, hgp_pins *out);
HGP_API void hgp_pins_free(hgp_ctx *ctx, hgp_pins *pm);

/* f1: Eq.1, Eq.16 and the loads of part (e.g. rho of hgp_coarsen on level 0).
 * part_size / part_inbound: DEVICE u64 [nparts] receiving every partition's loads, or NULL. */
HGP_API hgp_status hgp_partition_metrics(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                         uint64_t omega, uint64_t delta, hgp_quality *out, uint64_t *part_size,
                                         uint64_t *part_inbound);

/* f3: Eq.13: saving(n) = sum of omega(e) over e in I(n) with
 * pins(rho(n), e) = 1; loss(n, p) = sum of omega(e) over e in I(n) with pins(p, e) = 0;
 * dest[n] = the p != rho(n) holding a pin of some e in I(n) with the largest (gain(n, p), p),
 * restricted to size(n) + |p| <= omega when enforce_size; HGP_NONE (gain 0) if none.
 * pins: the full matrix from hgp_pins_matrix(part, inbound = 0), or NULL (computed here).
 * dest: DEVICE u32 [N]; gain: DEVICE i64 [N]. */
HGP_API hgp_status hgp_propose_moves(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                     const hgp_pins *pins, uint64_t omega, int enforce_size, uint32_t *dest,
                                     int64_t *gain);

/* f3: in-sequence gains (Eqs.14-15). seq: DEVICE [M] distinct node ids, each with
 * dest[n] < nparts and != part[n] (else HGP_E_ARG naming the lowest bad position); gain_seq[i]
 * (DEVICE i64 [M]) = Eq.1 before move i minus Eq.1 after it, moves 0..i-1 applied.
 * pins: full matrix of part, or NULL. */
HGP_API hgp_status hgp_in_sequence_gains(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                         const hgp_pins *pins, const uint32_t *seq, uint32_t M,
                                         const uint32_t *dest, int64_t *gain_seq);

/* f4: event-based constraint checks: violations[i] (DEVICE u32 [M]) = number of
 * partitions with size > omega or mu-weighted inbound load > delta after moves 0..i.
 * pins_in: the inbound matrix of part (hgp_pins_matrix(inbound = 1)), or NULL. */
HGP_API hgp_status hgp_sequence_violations(hgp_ctx *ctx, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                           const hgp_pins *pins_in, const uint32_t *seq, uint32_t M,
                                           const uint32_t *dest, uint64_t omega, uint64_t delta,
                                           uint32_t *violations);

/* f4: the landing point: *k (HOST) = the prefix length 1..M with violations[k-1]
 * = 0 and the largest cumulative in-sequence gain *best (HOST), the shortest on ties; k = 0 and
 * best = 0 when no such prefix has a gain > 0. gain_seq, violations: DEVICE [M]. */
HGP_API hgp_status hgp_best_prefix(hgp_ctx *ctx, const int64_t *gain_seq, const uint32_t *violations, uint32_t M,
                                   uint32_t *k, int64_t *best);

HGP_API void hgp_csr_free(hgp_ctx *ctx, hgp_csr *g);
HGP_API void hgp_nbrs_free(hgp_ctx *ctx, hgp_nbrs *nb);

#ifdef __cplusplus
}
#endif
#endif /* HGP_H */
