// hgp_ref.cpp — CPU ORACLE for one coarsening level (arXiv 2605.20497 §5).
//
// TEST INFRASTRUCTURE (see hgp_ref.h): plain, slow, single-threaded, shares no
// code with the CUDA path. Each function cites the passage it follows.
// Readings of silent/ambiguous passages refer to DESIGN.md "Readings" #n.
#include "hgp_ref.h"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

template <class T>
T *to_malloc(const std::vector<T> &v) {
  T *p = static_cast<T *>(malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
  if (p && !v.empty()) memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

const uint64_t kFp = HGP_REF_FP_SHIFT;

// ---------------------------------------------------------------------------
// Compressed sparse level: hyperedge segments with sources first,
// incidence segments with inbound edges first, plus |src(e)| and |in(n)|.
// ---------------------------------------------------------------------------
struct Level {
  uint32_t N = 0, E = 0;
  std::vector<uint64_t> edge_off;   // [E+1]
  std::vector<uint32_t> edge_nsrc;  // [E]
  std::vector<uint32_t> pins;       // src(e) ascending ‖ dst(e) ascending
  std::vector<uint32_t> edge_w, edge_mu, node_w;
};

// in(n) = {e : n in dst(e)}, out(n) = {e : n in src(e)}, stored in-first
// (P:493-495); each sub-list ascending by edge id (reading #15). Visiting edges
// in ascending order and appending yields ascending lists directly.
void build_incidence(const Level &L, std::vector<uint64_t> &inc_off, std::vector<uint32_t> &inc_nin,
                     std::vector<uint32_t> &inc, std::vector<uint32_t> &in_mu) {
  std::vector<std::vector<uint32_t>> in_l(L.N), out_l(L.N);
  for (uint32_t e = 0; e < L.E; ++e) {
    uint64_t lo = L.edge_off[e], hi = L.edge_off[e + 1], s = lo + L.edge_nsrc[e];
    for (uint64_t j = lo; j < hi; ++j) (j < s ? out_l : in_l)[L.pins[j]].push_back(e);
  }
  inc_off.assign(L.N + 1, 0);
  inc_nin.assign(L.N, 0);
  in_mu.assign(L.N, 0);
  inc.clear();
  for (uint32_t n = 0; n < L.N; ++n) {
    inc_nin[n] = static_cast<uint32_t>(in_l[n].size());
    uint64_t mu = 0;
    for (uint32_t e : in_l[n]) mu += L.edge_mu[e];
    in_mu[n] = static_cast<uint32_t>(mu);
    inc.insert(inc.end(), in_l[n].begin(), in_l[n].end());
    inc.insert(inc.end(), out_l[n].begin(), out_l[n].end());
    inc_off[n + 1] = inc.size();
  }
}

int export_level(const Level &L, hgp_ref_csr *out) {
  std::vector<uint64_t> inc_off;
  std::vector<uint32_t> inc_nin, inc, in_mu;
  build_incidence(L, inc_off, inc_nin, inc, in_mu);
  out->N = L.N;
  out->E = L.E;
  out->P = L.pins.size();
  out->edge_off = to_malloc(L.edge_off);
  out->edge_nsrc = to_malloc(L.edge_nsrc);
  out->pins = to_malloc(L.pins);
  out->edge_w = to_malloc(L.edge_w);
  out->edge_mu = to_malloc(L.edge_mu);
  out->node_w = to_malloc(L.node_w);
  out->inc_off = to_malloc(inc_off);
  out->inc_nin = to_malloc(inc_nin);
  out->inc = to_malloc(inc);
  out->in_mu = to_malloc(in_mu);
  if (!out->edge_off || !out->pins || !out->inc) return fail(HGP_REF_E_OOM, "out of host memory");
  return HGP_REF_OK;
}

// splitmix64 output function (Steele et al.), used as the "deterministic noise"
// hash of P:663-664 (reading #3).
uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

const char *hgp_ref_last_error(void) { return g_err.c_str(); }

void hgp_ref_csr_free(hgp_ref_csr *g) {
  if (!g) return;
  free(g->edge_off); free(g->edge_nsrc); free(g->pins); free(g->edge_w); free(g->edge_mu);
  free(g->node_w); free(g->inc_off); free(g->inc_nin); free(g->inc); free(g->in_mu);
  memset(g, 0, sizeof(*g));
}

void hgp_ref_nbrs_free(hgp_ref_nbrs *nb) {
  if (!nb) return;
  free(nb->off); free(nb->nbr);
  memset(nb, 0, sizeof(*nb));
}

// ---------------------------------------------------------------------------
// a1 — CSR materialisation (problem model P:290-297).
// Validation order (first failing category wins, lowest index inside it):
//   A structure of offsets, B pin range, C duplicate pins / src∩dst,
//   D omega = 0, E size = 0, F overflow guards (reading #2, #18).
// ---------------------------------------------------------------------------
int hgp_ref_build_csr(const hgp_ref_input *in, hgp_ref_csr *out) {
  if (!in || !out) return fail(HGP_REF_E_ARG, "null argument");
  memset(out, 0, sizeof(*out));
  const uint32_t N = in->num_nodes, E = in->num_edges;
  if (N >= (1u << 31)) return fail(HGP_REF_E_OVERFLOW, "num_nodes %u >= 2^31", N);
  if (E == HGP_REF_NONE) return fail(HGP_REF_E_OVERFLOW, "num_edges too large");
  if (in->edge_off[0] != 0) return fail(HGP_REF_E_MALFORMED, "edge 0: edge_off[0] != 0");
  // A: offsets monotone, edges non-empty, nsrc <= |e|, |e| <= 2^24
  for (uint32_t e = 0; e < E; ++e) {
    uint64_t lo = in->edge_off[e], hi = in->edge_off[e + 1];
    if (hi < lo) return fail(HGP_REF_E_MALFORMED, "edge %u: offsets decrease", e);
    if (hi == lo) return fail(HGP_REF_E_MALFORMED, "edge %u: empty hyperedge", e);
    if (in->edge_nsrc[e] > hi - lo) return fail(HGP_REF_E_MALFORMED, "edge %u: nsrc > |e|", e);
    if (hi - lo > (1ull << 24)) return fail(HGP_REF_E_OVERFLOW, "edge %u: |e| > 2^24", e);
  }
  const uint64_t P = E ? in->edge_off[E] : 0;
  // B: every pin is a node id
  for (uint32_t e = 0; e < E; ++e)
    for (uint64_t j = in->edge_off[e]; j < in->edge_off[e + 1]; ++j)
      if (in->pins[j] >= N) return fail(HGP_REF_E_MALFORMED, "edge %u: pin out of range", e);
  // Canonical edge: src(e) ascending, then dst(e) ascending (reading #15).
  Level L;
  L.N = N;
  L.E = E;
  L.edge_off.assign(in->edge_off, in->edge_off + E + 1);
  L.edge_nsrc.assign(in->edge_nsrc, in->edge_nsrc + E);
  L.pins.assign(in->pins, in->pins + P);
  for (uint32_t e = 0; e < E; ++e) {
    uint32_t *b = L.pins.data() + L.edge_off[e];
    uint32_t *s = b + L.edge_nsrc[e];
    uint32_t *x = L.pins.data() + L.edge_off[e + 1];
    std::sort(b, s);
    std::sort(s, x);
  }
  // C: "no duplicate pins nor self-cycles, src(e) ∩ dst(e) = ∅"
  for (uint32_t e = 0; e < E; ++e) {
    std::vector<uint32_t> all(L.pins.begin() + L.edge_off[e], L.pins.begin() + L.edge_off[e + 1]);
    std::sort(all.begin(), all.end());
    if (std::adjacent_find(all.begin(), all.end()) != all.end())
      return fail(HGP_REF_E_MALFORMED, "edge %u: duplicate pin", e);
  }
  // D, E: positive weights and sizes
  for (uint32_t e = 0; e < E; ++e)
    if (in->edge_w[e] == 0) return fail(HGP_REF_E_MALFORMED, "edge %u: zero weight", e);
  for (uint32_t n = 0; n < N; ++n)
    if (in->node_w[n] == 0) return fail(HGP_REF_E_MALFORMED, "node %u: zero size", n);
  // F: sum omega < 2^32 and sum size < 2^32 (reading #2, #18)
  uint64_t sw = 0, sn = 0;
  for (uint32_t e = 0; e < E; ++e) sw += in->edge_w[e];
  for (uint32_t n = 0; n < N; ++n) sn += in->node_w[n];
  if (sw >= (1ull << 32)) return fail(HGP_REF_E_OVERFLOW, "sum of edge weights >= 2^32");
  if (sn >= (1ull << 32)) return fail(HGP_REF_E_OVERFLOW, "sum of node sizes >= 2^32");
  L.edge_w.assign(in->edge_w, in->edge_w + E);
  L.edge_mu.assign(E, 1u);  // level 0: every edge stands for one original edge (reading #12)
  L.node_w.assign(in->node_w, in->node_w + N);
  return export_level(L, out);
}

// ---------------------------------------------------------------------------
// a2 — unique neighbourhoods: N(n) = {m in e | e in I(n)} \ {n},
// materialised once, ascending, purge bits clear.
// ---------------------------------------------------------------------------
int hgp_ref_unique_neighbors(const hgp_ref_csr *g, uint32_t lo, uint32_t hi, hgp_ref_nbrs *out) {
  if (!g || !out || lo > hi || hi > g->N) return fail(HGP_REF_E_ARG, "bad node range");
  memset(out, 0, sizeof(*out));
  std::vector<uint64_t> off(1, 0);
  std::vector<uint32_t> nbr;
  for (uint32_t n = lo; n < hi; ++n) {
    std::vector<uint32_t> s;
    for (uint64_t k = g->inc_off[n]; k < g->inc_off[n + 1]; ++k) {
      uint32_t e = g->inc[k];
      for (uint64_t j = g->edge_off[e]; j < g->edge_off[e + 1]; ++j)
        if (g->pins[j] != n) s.push_back(g->pins[j]);
    }
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    nbr.insert(nbr.end(), s.begin(), s.end());
    off.push_back(nbr.size());
  }
  out->lo = lo;
  out->hi = hi;
  out->V = nbr.size();
  out->off = to_malloc(off);
  out->nbr = to_malloc(nbr);
  return HGP_REF_OK;
}

// ---------------------------------------------------------------------------
// a3 — candidate pairs proposal (§5.3; Eqs.5-6; top-Pi P:770-771).
// Integer fixed point (reading #2): c(e) = floor(omega(e) * 2^24 / |e|) (Eq.5),
// or omega(e) * 2^24 with norm = 1 (reading #1).
// ---------------------------------------------------------------------------
int hgp_ref_score_pairs(const hgp_ref_csr *g, hgp_ref_nbrs *nb, const hgp_ref_params *p,
                        hgp_ref_cand *cand) {
  if (!g || !nb || !p || !cand) return fail(HGP_REF_E_ARG, "null argument");
  if (p->pi < 1 || p->pi > 16) return fail(HGP_REF_E_ARG, "pi must be in [1,16]");
  if (p->norm > 1) return fail(HGP_REF_E_ARG, "norm must be 0 or 1");
  if (p->noise_cap >= (1ull << 56)) return fail(HGP_REF_E_ARG, "noise_cap >= 2^56");
  if (nb->hi > g->N || nb->lo > nb->hi) return fail(HGP_REF_E_ARG, "bad neighbour range");
  const uint32_t pi = p->pi;
  // Overflow guard (reading #2): every matching total stays below 2^62.
  {
    unsigned __int128 tot = 0;
    for (uint32_t e = 0; e < g->E; ++e) {
      uint64_t sz = g->edge_off[e + 1] - g->edge_off[e];
      tot += (unsigned __int128)(p->norm ? sz : 1) * g->edge_w[e];
    }
    tot <<= kFp;
    tot += (unsigned __int128)(g->N / 2 + 1) * p->noise_cap;
    if (tot >= ((unsigned __int128)1 << 62)) return fail(HGP_REF_E_OVERFLOW, "score totals may exceed 2^62");
  }
  // A valid solution is assumed to exist: every node alone must fit.
  for (uint32_t n = nb->lo; n < nb->hi; ++n) {
    if (g->node_w[n] > p->omega) return fail(HGP_REF_E_INFEASIBLE, "node %u: size exceeds omega", n);
    if (p->delta != HGP_REF_UNBOUNDED && g->in_mu[n] > p->delta)
      return fail(HGP_REF_E_INFEASIBLE, "node %u: inbound edges exceed delta", n);
  }
  const uint64_t seed_mix = splitmix64(p->noise_seed);
  auto c_of = [&](uint32_t e) -> uint64_t {                       // Eq.5 weight term
    uint64_t w = static_cast<uint64_t>(g->edge_w[e]) << kFp;
    return p->norm ? w : w / (g->edge_off[e + 1] - g->edge_off[e]);
  };
  auto noise = [&](uint32_t n, uint32_t m) -> uint64_t {          // rng(min(n,m), max(n,m))
    if (p->noise_cap == 0) return 0;
    uint64_t key = (static_cast<uint64_t>(std::min(n, m)) << 32) | std::max(n, m);
    // uniform in [0, cap]: floor(hash * (cap + 1) / 2^64) (reading #3)
    return static_cast<uint64_t>(((unsigned __int128)splitmix64(key ^ seed_mix) * (p->noise_cap + 1)) >> 64);
  };
  struct Bin { uint32_t id; uint64_t pos; uint64_t eta; uint64_t inter; };
  for (uint32_t n = nb->lo; n < nb->hi; ++n) {
    const uint64_t b0 = nb->off[n - nb->lo], b1 = nb->off[n - nb->lo + 1];
    // Neighbours still eligible: purge bit clear.
    std::vector<uint64_t> live;
    for (uint64_t k = b0; k < b1; ++k)
      if (!(nb->nbr[k] & HGP_REF_PURGE)) live.push_back(k);
    const uint64_t B = p->batch ? p->batch : (live.empty() ? 1 : live.size());
    std::vector<std::pair<uint64_t, uint32_t>> top;  // (score, id), best first
    // "we load a fixed-size batch of them at once ... repeated for all neighbor batches"
    for (uint64_t bs = 0; bs < live.size(); bs += B) {
      std::vector<Bin> bins;                                     // sorted by id
      for (uint64_t k = bs; k < std::min<uint64_t>(bs + B, live.size()); ++k)
        bins.push_back({nb->nbr[live[k]], live[k], 0, 0});
      // Visit I(n) (in-edges first) and every pin; binary search for the bin.
      for (uint64_t k = g->inc_off[n]; k < g->inc_off[n + 1]; ++k) {
        const uint32_t e = g->inc[k];
        const bool e_in = k < g->inc_off[n] + g->inc_nin[n];     // e in in(n)
        const uint64_t lo = g->edge_off[e], s = lo + g->edge_nsrc[e], hi = g->edge_off[e + 1];
        for (uint64_t j = lo; j < hi; ++j) {
          const uint32_t m = g->pins[j];
          if (m == n) continue;
          auto it = std::lower_bound(bins.begin(), bins.end(), m,
                                     [](const Bin &b, uint32_t v) { return b.id < v; });
          if (it == bins.end() || it->id != m) continue;         // m in another batch
          it->eta += c_of(e);                                    // Eq.5
          if (e_in && j >= s) it->inter += g->edge_mu[e];        // m in dst(e), e in in(n)
        }
      }
      // Noise, validity (Eq.6, P:535 with P:623), purge flags on every invalid bin (reading #6).
      std::vector<std::pair<uint64_t, uint32_t>> valid;
      for (Bin &b : bins) {
        b.eta += noise(n, b.id);
        const bool size_ok = static_cast<uint64_t>(g->node_w[n]) + g->node_w[b.id] <= p->omega;
        const uint64_t uni = static_cast<uint64_t>(g->in_mu[n]) + g->in_mu[b.id] - b.inter;  // |in(n) ∪ in(m)|
        const bool in_ok = p->delta == HGP_REF_UNBOUNDED || uni <= p->delta;
        if (size_ok && in_ok) valid.push_back({b.eta, b.id});
        else nb->nbr[b.pos] |= HGP_REF_PURGE;
      }
      // Sort by (eta desc, id desc) — max_id argmax (Eq.6) — and keep the best Pi.
      std::sort(valid.begin(), valid.end(), [](const auto &x, const auto &y) {
        return x.first != y.first ? x.first > y.first : x.second > y.second;
      });
      top.insert(top.end(), valid.begin(), valid.end());
      std::sort(top.begin(), top.end(), [](const auto &x, const auto &y) {
        return x.first != y.first ? x.first > y.first : x.second > y.second;
      });
      if (top.size() > pi) top.resize(pi);
    }
    for (uint32_t i = 0; i < pi; ++i) {
      hgp_ref_cand &c = cand[static_cast<uint64_t>(n) * pi + i];
      c.pad = 0;
      if (i < top.size()) { c.id = top[i].second; c.score = top[i].first; }
      else { c.id = HGP_REF_NONE; c.score = 0; }
    }
  }
  return HGP_REF_OK;
}

// ---------------------------------------------------------------------------
// a4 — maximum-weight matching on the two-cycle pseudo-forest (§5.4, Eqs.7-12,
// P:679-741), repeated over Pi proposal graphs with removal.
// ---------------------------------------------------------------------------
int hgp_ref_match(const hgp_ref_cand *cand, uint32_t N, uint32_t pi, uint32_t *match,
                  uint32_t *matched_per_round, int64_t *round_value) {
  if ((!cand && N) || (!match && N) || pi < 1 || pi > 16) return fail(HGP_REF_E_ARG, "bad argument");
  const uint32_t NONE = HGP_REF_NONE;
  const int64_t NEG_INF = INT64_MIN;
  for (uint32_t n = 0; n < N; ++n) match[n] = NONE;
  std::vector<char> matched(N, 0);
  for (uint32_t i = 0; i < pi; ++i) {
    // target / score of round i; nodes matched earlier are removed
    std::vector<uint32_t> t(N, NONE);
    std::vector<int64_t> s(N, 0);
    for (uint32_t n = 0; n < N; ++n) {
      const hgp_ref_cand &c = cand[static_cast<uint64_t>(n) * pi + i];
      if (c.id != NONE && c.id >= N) return fail(HGP_REF_E_ARG, "node %u: candidate id out of range", n);
      if (!matched[n] && c.id != NONE && !matched[c.id]) { t[n] = c.id; s[n] = static_cast<int64_t>(c.score); }
    }
    // R = {n | target(target(n)) = n}; child(n) = {c | target(c) = n} \ R
    std::vector<char> inR(N, 0);
    for (uint32_t n = 0; n < N; ++n)
      if (t[n] != NONE && t[t[n]] == n) inR[n] = 1;
    std::vector<std::vector<uint32_t>> child(N);
    for (uint32_t c = 0; c < N; ++c)
      if (t[c] != NONE && !inR[c]) child[t[c]].push_back(c);
    // Post-order over each pseudo-tree from its roots: the pairs in R and nodes with no target.
    std::vector<uint32_t> order;
    std::vector<char> seen(N, 0);
    for (uint32_t r = 0; r < N; ++r) {
      if (!(inR[r] || t[r] == NONE) || seen[r]) continue;
      std::vector<std::pair<uint32_t, size_t>> st{{r, 0}};
      seen[r] = 1;
      while (!st.empty()) {
        auto &top = st.back();
        if (top.second < child[top.first].size()) {
          uint32_t c = child[top.first][top.second++];
          seen[c] = 1;
          st.push_back({c, 0});
        } else {
          order.push_back(top.first);
          st.pop_back();
        }
      }
    }
    for (uint32_t n = 0; n < N; ++n)
      if (!seen[n]) return fail(HGP_REF_E_INTERNAL, "round %u: node %u lies on a proposal cycle longer than 2", i, n);
    std::vector<int64_t> ss0(N, 0), ss1(N, NEG_INF), sum0(N, 0);
    std::vector<uint32_t> best(N, NONE);   // argmax_c ss_{1-0}(c), kept only when the max is > 0
    for (uint32_t n : order) {
      int64_t g = 0;
      bool any = false;
      uint32_t arg = NONE;
      for (uint32_t c : child[n]) {
        sum0[n] += ss0[c];
        const int64_t d = ss1[c] - ss0[c];                         // ss_{1-0}(c)
        if (!any || d > g || (d == g && c > arg)) { g = d; arg = c; any = true; }
      }
      ss0[n] = sum0[n] + (any && g > 0 ? g : 0);                   // Eq.10
      if (any && g > 0) best[n] = arg;
      if (t[n] != NONE && !inR[n]) ss1[n] = s[n] + sum0[n];        // Eq.7
    }
    // Roots (Eq.8, Eq.11): decide each mutual pair once, on its lower id (reading #9).
    int64_t value = 0;
    for (uint32_t r = 0; r < N; ++r) {
      if (t[r] == NONE) { value += ss0[r]; continue; }
      if (!inR[r] || r > t[r]) continue;
      const uint32_t q = t[r];
      if (s[r] != s[q]) return fail(HGP_REF_E_INTERNAL, "round %u: asymmetric scores on pair %u-%u", i, r, q);
      ss1[r] = ss1[q] = s[r] + sum0[r] + sum0[q];                  // Eq.8
      if (ss1[r] > ss0[r] + ss0[q]) { match[r] = q; match[q] = r; value += ss1[r]; }
      else {
        value += ss0[r] + ss0[q];
        if (best[r] != NONE) match[r] = best[r];                   // Eq.11 second branch + > 0 guard
        if (best[q] != NONE) match[q] = best[q];
      }
    }
    // Top-down (Eq.12): parents before children = reverse post-order.
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      const uint32_t n = *it;
      if (inR[n]) continue;
      if (t[n] == NONE) {                                          // terminal: only children can match it
        if (best[n] != NONE) match[n] = best[n];
        continue;
      }
      if (match[t[n]] == n) match[n] = t[n];                       // Eq.12 first branch
      else if (best[n] != NONE) match[n] = best[n];                // Eq.12 second branch
      else match[n] = NONE;                                        // Eq.12 third branch
    }
    uint32_t pairs = 0;
    for (uint32_t n = 0; n < N; ++n) {
      if (matched[n] || match[n] == NONE) continue;
      if (match[match[n]] != n) return fail(HGP_REF_E_INTERNAL, "round %u: asymmetric match at %u", i, n);
      if (n < match[n]) ++pairs;
    }
    for (uint32_t n = 0; n < N; ++n)
      if (match[n] != NONE) matched[n] = 1;
    if (matched_per_round) matched_per_round[i] = pairs;
    if (round_value) round_value[i] = value;
  }
  return HGP_REF_OK;
}

// ---------------------------------------------------------------------------
// a5 — coarse hypergraph construction (§5.5; §3).
// ---------------------------------------------------------------------------
int hgp_ref_contract(const hgp_ref_csr *g, const hgp_ref_nbrs *nb, const uint32_t *match,
                     uint32_t *gamma, hgp_ref_csr *coarse, hgp_ref_nbrs *coarse_nb) {
  if (!g || !nb || !match || !gamma || !coarse || !coarse_nb) return fail(HGP_REF_E_ARG, "null argument");
  if (nb->lo != 0 || nb->hi != g->N) return fail(HGP_REF_E_ARG, "contract needs neighbours of every node");
  const uint32_t N = g->N, NONE = HGP_REF_NONE;
  for (uint32_t n = 0; n < N; ++n)
    if (match[n] != NONE && (match[n] >= N || match[n] == n || match[match[n]] != n))
      return fail(HGP_REF_E_ARG, "node %u: match is not symmetric", n);
  // gamma(n) = {n, match(n)}; coarse ids by ascending min member (reading #11).
  std::vector<uint32_t> cid(N, NONE);
  uint32_t Nc = 0;
  for (uint32_t n = 0; n < N; ++n)
    if (match[n] == NONE || n < match[n]) cid[n] = Nc++;
  for (uint32_t n = 0; n < N; ++n) gamma[n] = cid[match[n] == NONE ? n : std::min(n, match[n])];
  Level C;
  C.N = Nc;
  C.node_w.assign(Nc, 0);
  for (uint32_t n = 0; n < N; ++n) C.node_w[gamma[n]] += g->node_w[n];  // size(n') = sum
  // E' = {{gamma(n) | n in e}}; src/dst duplicates are kept in dst;
  // drop iff D' empty and |S'| <= 1 (reading #14); parallel edges merged (reading #12).
  std::map<std::pair<std::vector<uint32_t>, std::vector<uint32_t>>, uint32_t> cls;
  C.edge_off.push_back(0);
  for (uint32_t e = 0; e < g->E; ++e) {
    const uint64_t lo = g->edge_off[e], s = lo + g->edge_nsrc[e], hi = g->edge_off[e + 1];
    std::vector<uint32_t> D, S;
    for (uint64_t j = s; j < hi; ++j) D.push_back(gamma[g->pins[j]]);
    std::sort(D.begin(), D.end());
    D.erase(std::unique(D.begin(), D.end()), D.end());
    for (uint64_t j = lo; j < s; ++j) {
      const uint32_t x = gamma[g->pins[j]];
      if (!std::binary_search(D.begin(), D.end(), x)) S.push_back(x);
    }
    std::sort(S.begin(), S.end());
    S.erase(std::unique(S.begin(), S.end()), S.end());
    if (D.empty() && S.size() <= 1) continue;
    auto key = std::make_pair(S, D);
    auto it = cls.find(key);
    if (it == cls.end()) {                                           // representative = min edge id
      cls.emplace(key, C.E);
      C.edge_nsrc.push_back(static_cast<uint32_t>(S.size()));
      C.pins.insert(C.pins.end(), S.begin(), S.end());
      C.pins.insert(C.pins.end(), D.begin(), D.end());
      C.edge_off.push_back(C.pins.size());
      C.edge_w.push_back(g->edge_w[e]);
      C.edge_mu.push_back(g->edge_mu[e]);
      ++C.E;
    } else {                                                         // omega' = sum omega, mu' = sum mu
      C.edge_w[it->second] += g->edge_w[e];
      C.edge_mu[it->second] += g->edge_mu[e];
    }
  }
  memset(coarse, 0, sizeof(*coarse));
  int rc = export_level(C, coarse);
  if (rc) return rc;
  // N'(c) = gamma(N(a) ∪ N(b)) minus entries flagged anywhere (OR; reading #7),
  // minus c itself; flags cleared (reading #16).
  std::vector<std::vector<uint32_t>> members(Nc);
  for (uint32_t n = 0; n < N; ++n) members[gamma[n]].push_back(n);
  std::vector<uint64_t> off(1, 0);
  std::vector<uint32_t> nbr;
  for (uint32_t c = 0; c < Nc; ++c) {
    std::vector<uint32_t> X, F;
    for (uint32_t a : members[c])
      for (uint64_t k = nb->off[a]; k < nb->off[a + 1]; ++k) {
        const uint32_t v = nb->nbr[k];
        const uint32_t gm = gamma[v & ~HGP_REF_PURGE];
        X.push_back(gm);
        if (v & HGP_REF_PURGE) F.push_back(gm);
      }
    std::sort(X.begin(), X.end());
    X.erase(std::unique(X.begin(), X.end()), X.end());
    std::sort(F.begin(), F.end());
    for (uint32_t x : X)
      if (x != c && !std::binary_search(F.begin(), F.end(), x)) nbr.push_back(x);
    off.push_back(nbr.size());
  }
  memset(coarse_nb, 0, sizeof(*coarse_nb));
  coarse_nb->lo = 0;
  coarse_nb->hi = Nc;
  coarse_nb->V = nbr.size();
  coarse_nb->off = to_malloc(off);
  coarse_nb->nbr = to_malloc(nbr);
  return HGP_REF_OK;
}

int hgp_ref_coarsen_level(const hgp_ref_csr *g, hgp_ref_nbrs *nb, const hgp_ref_params *p,
                          hgp_ref_cand *cand, uint32_t *match, uint32_t *gamma, hgp_ref_csr *coarse,
                          hgp_ref_nbrs *coarse_nb) {
  if (!g || !nb || nb->lo != 0 || nb->hi != g->N) return fail(HGP_REF_E_ARG, "level needs all neighbours");
  int rc = hgp_ref_score_pairs(g, nb, p, cand);
  if (rc) return rc;
  rc = hgp_ref_match(cand, g->N, p->pi, match, nullptr, nullptr);
  if (rc) return rc;
  return hgp_ref_contract(g, nb, match, gamma, coarse, coarse_nb);
}

}  // extern "C"

// error reporting for the next-row functions (hgp_ref_refine.cpp)
int hgp_ref_set_error(int code, const char *msg) { return fail(code, "%s", msg); }
