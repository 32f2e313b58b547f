/* hgpgen — seeded synthetic directed-hypergraph generators.
 *
 * This module is shared by the CPU oracle (oracle/) and the CUDA path
 * (paper_2605_20497_b200/) ONLY as a source of inputs. It holds none of the
 * method's arithmetic: it draws hypergraphs (pins, weights) and nothing else.
 * Recipes follow SURVEY.md §8(d) and are restated in DESIGN.md §"Input recipe".
 *
 * All arrays are malloc'd by the generator and released with hgpgen_free().
 * Random numbers: xoshiro256** seeded through splitmix64 (Blackman & Vigna).
 */
#ifndef HGPGEN_H
#define HGPGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t num_nodes, num_edges;
  uint64_t num_pins;
  uint64_t *edge_off;   /* [E+1] */
  uint32_t *edge_nsrc;  /* [E]   first nsrc pins of a segment are sources       */
  uint32_t *pins;       /* [P]   unsorted inside the src / dst blocks           */
  uint32_t *edge_w;     /* [E]   omega(e) >= 1                                   */
  uint32_t *node_w;     /* [N]   size(n) >= 1                                    */
} hgpgen_graph;

/* C1 "tiny": |e| = 2 + Binomial(12, 1/2); nsrc = 1 (p .8), 0 (p .1), 2 (p .1);
 * pins uniform without replacement; omega ~ U{1..wmax_e}; size(n) = 1 or U{1..wmax_n};
 * destination draws resampled so that |in(n)| <= in_cap. */
int hgpgen_tiny(uint64_t seed, uint32_t num_nodes, uint32_t num_edges, uint32_t size_base,
                uint32_t size_binom, uint32_t in_cap, uint32_t wmax_e, uint32_t wmax_n,
                hgpgen_graph *out);

/* C2/C5 "SNN-mapping": layers x rows x cols neurons; neuron n owns one axon
 * hyperedge src{n} + fanout distinct destinations of layer (l+1) mod L drawn
 * from the window x window patch around n's coordinates (clamped to the grid);
 * each destination is rewired with probability rewire to a uniform neuron of
 * that layer ("-rand").  omega = 1, size = 1. */
int hgpgen_snn(uint64_t seed, uint32_t layers, uint32_t rows, uint32_t cols, uint32_t fanout,
               uint32_t window, double rewire, hgpgen_graph *out);

/* C3/C4 "VLSI-like": |e| ~ discrete power law on [dmin, dmax] with exponent alpha;
 * one driver (src) per net, uniform; each sink with probability locality from a
 * window of width 16|e| around the driver id, else Zipf(1) over a seeded node
 * permutation (hubs); |in(n)| capped at in_cap by resampling. omega = 1, size = 1. */
int hgpgen_vlsi(uint64_t seed, uint32_t num_nodes, uint32_t num_edges, uint32_t dmin,
                uint32_t dmax, double alpha, double locality, uint32_t in_cap,
                hgpgen_graph *out);

void hgpgen_free(hgpgen_graph *g);

#ifdef __cplusplus
}
#endif
#endif
