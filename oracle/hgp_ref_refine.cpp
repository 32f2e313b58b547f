// hgp_ref_refine.cpp — CPU ORACLE for the rows after the level: the quality of a
// partition (f1), refinement gains (f3) and the validation of a move sequence (f4).
//
// TEST INFRASTRUCTURE (see hgp_ref.h): plain, slow, single-threaded, shares no code with the
// CUDA path. Every result here has a plain definition, so each function IS that definition
// written out (std::map / std::set per hyperedge, sequential simulation of the moves), not the
// paper's parallel algorithm:
//  - Eq.1 connectivity, Eq.16 cut-net, the size and distinct-inbound
//    counts of every partition (inbound counts mu-weighted, reading #12);
//  - pins(p, e) / pins_in(p, e);
//  - Eq.13 saving / loss / gain and the proposed move;
//  - the in-sequence gain of a move = the connectivity change it causes when every
//    earlier move of the sequence is already applied (the property S:410 states exactly);
//  - the number of violated constraints after each move by replaying the moves.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <vector>

#include "hgp_ref.h"

int hgp_ref_set_error(int code, const char *msg);

namespace {

struct View {   // the level's edges as (src set, dst set) and incidence I(n)
  const hgp_ref_csr *g;
  uint64_t lo(uint32_t e) const { return g->edge_off[e]; }
  uint64_t hi(uint32_t e) const { return g->edge_off[e + 1]; }
  uint64_t ds(uint32_t e) const { return g->edge_off[e] + g->edge_nsrc[e]; }   // first dst pin
};

int check_part(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts) {
  if (!g || (g->N && !part)) return hgp_ref_set_error(HGP_REF_E_ARG, "null argument");
  for (uint32_t n = 0; n < g->N; ++n)
    if (part[n] >= nparts) return hgp_ref_set_error(HGP_REF_E_ARG, "partition id out of range");
  return HGP_REF_OK;
}

// connectivity contribution of edge e under the per-partition pin counts `cnt` (Eq.1)
uint64_t lambda_of(const std::map<uint32_t, int64_t> &cnt) {
  uint64_t l = 0;
  for (const auto &kv : cnt) l += kv.second > 0;
  return l;
}

int check_seq(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, const uint32_t *seq, uint32_t M,
              const uint32_t *dest) {
  int rc = check_part(g, part, nparts);
  if (rc) return rc;
  if (M && (!seq || !dest)) return hgp_ref_set_error(HGP_REF_E_ARG, "null sequence");
  std::vector<char> seen(g->N, 0);
  for (uint32_t i = 0; i < M; ++i) {
    const uint32_t n = seq[i];
    if (n >= g->N || seen[n]) return hgp_ref_set_error(HGP_REF_E_ARG, "sequence entries must be distinct nodes");
    seen[n] = 1;
    if (dest[n] >= nparts || dest[n] == part[n]) return hgp_ref_set_error(HGP_REF_E_ARG, "bad move destination");
  }
  return HGP_REF_OK;
}

}  // namespace

extern "C" {

// f1: Eq.1, Eq.16 and the constraint loads of the partition `part`.
int hgp_ref_partition_metrics(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, uint64_t omega,
                              uint64_t delta, hgp_ref_quality *out) {
  int rc = check_part(g, part, nparts);
  if (rc) return rc;
  if (!out) return hgp_ref_set_error(HGP_REF_E_ARG, "null output");
  View V{g};
  hgp_ref_quality q{};
  std::vector<uint64_t> size(nparts, 0), inb(nparts, 0);
  for (uint32_t n = 0; n < g->N; ++n) size[part[n]] += g->node_w[n];
  for (uint32_t e = 0; e < g->E; ++e) {
    std::set<uint32_t> lam, dparts;                       // {rho(n) | n in e}, {rho(n) | n in dst(e)}
    for (uint64_t j = V.lo(e); j < V.hi(e); ++j) lam.insert(part[g->pins[j]]);
    for (uint64_t j = V.ds(e); j < V.hi(e); ++j) dparts.insert(part[g->pins[j]]);
    q.connectivity += (uint64_t)g->edge_w[e] * (lam.size() - 1);
    if (lam.size() > 1) q.cut_net += g->edge_w[e];
    for (uint32_t p : dparts) inb[p] += g->edge_mu[e];    // e is inbound to p
  }
  for (uint32_t p = 0; p < nparts; ++p) {
    q.max_size = std::max(q.max_size, size[p]);
    q.max_inbound = std::max(q.max_inbound, inb[p]);
    if (size[p] > omega) ++q.size_violations;
    if (delta != HGP_REF_UNBOUNDED && inb[p] > delta) ++q.inbound_violations;
  }
  *out = q;
  return HGP_REF_OK;
}

// f3: pins(p, e) = |{n in e : rho(n) = p}|, pins_in(p, e) = |{n in dst(e) : rho(n) = p}|
int hgp_ref_pins_matrix(const hgp_ref_csr *g, const uint32_t *part, int inbound, hgp_ref_pins *out) {
  if (!g || !out || (g->N && !part)) return hgp_ref_set_error(HGP_REF_E_ARG, "null argument");
  View V{g};
  std::vector<uint64_t> off(1, 0);
  std::vector<uint32_t> pp, cc;
  for (uint32_t e = 0; e < g->E; ++e) {
    std::map<uint32_t, uint32_t> cnt;
    for (uint64_t j = inbound ? V.ds(e) : V.lo(e); j < V.hi(e); ++j) ++cnt[part[g->pins[j]]];
    for (const auto &kv : cnt) { pp.push_back(kv.first); cc.push_back(kv.second); }
    off.push_back(pp.size());
  }
  out->E = g->E;
  out->nnz = pp.size();
  out->off = static_cast<uint64_t *>(malloc(sizeof(uint64_t) * off.size()));
  out->part = static_cast<uint32_t *>(malloc(sizeof(uint32_t) * (pp.empty() ? 1 : pp.size())));
  out->count = static_cast<uint32_t *>(malloc(sizeof(uint32_t) * (cc.empty() ? 1 : cc.size())));
  memcpy(out->off, off.data(), sizeof(uint64_t) * off.size());
  if (!pp.empty()) {
    memcpy(out->part, pp.data(), sizeof(uint32_t) * pp.size());
    memcpy(out->count, cc.data(), sizeof(uint32_t) * cc.size());
  }
  return HGP_REF_OK;
}

void hgp_ref_pins_free(hgp_ref_pins *pm) {
  if (!pm) return;
  free(pm->off);
  free(pm->part);
  free(pm->count);
  memset(pm, 0, sizeof(*pm));
}

// f3: Eq.13 — saving(n) = sum over e in I(n) with pins(rho(n), e) = 1 of omega(e);
// loss(n, p) = sum over e in I(n) with pins(p, e) = 0 of omega(e); gain = saving - loss;
// move(n) = max_id argmax_p gain(n, p) over the partitions p != rho(n) holding a pin of some
// incident edge (S: propose_moves), restricted to size(n) + |p| <= Omega when enforce_size.
int hgp_ref_propose_moves(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, uint64_t omega,
                          int enforce_size, uint32_t *dest, int64_t *gain) {
  int rc = check_part(g, part, nparts);
  if (rc) return rc;
  if (g->N && (!dest || !gain)) return hgp_ref_set_error(HGP_REF_E_ARG, "null output");
  View V{g};
  std::vector<uint64_t> size(nparts, 0);
  for (uint32_t n = 0; n < g->N; ++n) size[part[n]] += g->node_w[n];
  std::vector<std::map<uint32_t, uint32_t>> pins(g->E);  // pins(p, e)
  for (uint32_t e = 0; e < g->E; ++e)
    for (uint64_t j = V.lo(e); j < V.hi(e); ++j) ++pins[e][part[g->pins[j]]];
  for (uint32_t n = 0; n < g->N; ++n) {
    const uint32_t ps = part[n];
    std::set<uint32_t> cands;                               // partitions holding a pin of I(n)
    int64_t saving = 0, total = 0;
    for (uint64_t k = g->inc_off[n]; k < g->inc_off[n + 1]; ++k) {
      const uint32_t e = g->inc[k];
      total += g->edge_w[e];
      if (pins[e].at(ps) == 1) saving += g->edge_w[e];
      for (const auto &kv : pins[e])
        if (kv.first != ps) cands.insert(kv.first);
    }
    uint32_t best = HGP_REF_NONE;
    int64_t bg = 0;
    for (uint32_t p : cands) {                              // ascending p: ties -> the larger id
      if (enforce_size && (uint64_t)g->node_w[n] + size[p] > omega) continue;
      int64_t loss = 0;
      for (uint64_t k = g->inc_off[n]; k < g->inc_off[n + 1]; ++k) {
        const uint32_t e = g->inc[k];
        if (!pins[e].count(p)) loss += g->edge_w[e];
      }
      const int64_t gp = saving - loss;
      if (best == HGP_REF_NONE || gp >= bg) { best = p; bg = gp; }
    }
    (void)total;
    dest[n] = best;
    gain[n] = best == HGP_REF_NONE ? 0 : bg;
  }
  return HGP_REF_OK;
}

// f3: the in-sequence gain by replaying the sequence: move i's gain is the
// connectivity (Eq.1) before it minus the connectivity after it, moves 0..i-1 applied.
int hgp_ref_in_sequence_gains(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, const uint32_t *seq,
                              uint32_t M, const uint32_t *dest, int64_t *gain_seq) {
  int rc = check_seq(g, part, nparts, seq, M, dest);
  if (rc) return rc;
  if (M && !gain_seq) return hgp_ref_set_error(HGP_REF_E_ARG, "null output");
  View V{g};
  std::vector<uint32_t> rho(part, part + g->N);
  std::vector<std::map<uint32_t, int64_t>> pins(g->E);
  for (uint32_t e = 0; e < g->E; ++e)
    for (uint64_t j = V.lo(e); j < V.hi(e); ++j) ++pins[e][rho[g->pins[j]]];
  for (uint32_t i = 0; i < M; ++i) {
    const uint32_t n = seq[i], ps = rho[n], pd = dest[n];
    int64_t before = 0, after = 0;
    for (uint64_t k = g->inc_off[n]; k < g->inc_off[n + 1]; ++k) {
      const uint32_t e = g->inc[k];
      before += (int64_t)g->edge_w[e] * (int64_t)(lambda_of(pins[e]) - 1);
      --pins[e][ps];
      ++pins[e][pd];
      after += (int64_t)g->edge_w[e] * (int64_t)(lambda_of(pins[e]) - 1);
    }
    rho[n] = pd;
    gain_seq[i] = before - after;
  }
  return HGP_REF_OK;
}

// f4: after each move of the sequence, how many partitions exceed Omega (size) or Delta (number
// of distinct inbound hyperedges, mu-weighted), by replaying the moves.
int hgp_ref_sequence_violations(const hgp_ref_csr *g, const uint32_t *part, uint32_t nparts, const uint32_t *seq,
                                uint32_t M, const uint32_t *dest, uint64_t omega, uint64_t delta,
                                uint32_t *violations) {
  int rc = check_seq(g, part, nparts, seq, M, dest);
  if (rc) return rc;
  if (M && !violations) return hgp_ref_set_error(HGP_REF_E_ARG, "null output");
  View V{g};
  std::vector<uint32_t> rho(part, part + g->N);
  std::vector<uint64_t> size(nparts, 0), inb(nparts, 0);
  std::vector<std::map<uint32_t, int64_t>> pins_in(g->E);   // pins_in(p, e)
  for (uint32_t n = 0; n < g->N; ++n) size[rho[n]] += g->node_w[n];
  for (uint32_t e = 0; e < g->E; ++e) {
    for (uint64_t j = V.ds(e); j < V.hi(e); ++j) ++pins_in[e][rho[g->pins[j]]];
    for (const auto &kv : pins_in[e]) inb[kv.first] += g->edge_mu[e];
  }
  auto bad = [&](uint32_t p) {
    return size[p] > omega || (delta != HGP_REF_UNBOUNDED && inb[p] > delta);
  };
  for (uint32_t i = 0; i < M; ++i) {
    const uint32_t n = seq[i], ps = rho[n], pd = dest[n];
    size[ps] -= g->node_w[n];
    size[pd] += g->node_w[n];
    const uint64_t i0 = g->inc_off[n], i1 = i0 + g->inc_nin[n];   // in(n)
    for (uint64_t k = i0; k < i1; ++k) {
      const uint32_t e = g->inc[k];
      if (--pins_in[e][ps] == 0) inb[ps] -= g->edge_mu[e];       // e no longer inbound to p_s
      if (++pins_in[e][pd] == 1) inb[pd] += g->edge_mu[e];       // e newly inbound to p_d
    }
    rho[n] = pd;
    uint32_t v = 0;
    for (uint32_t p = 0; p < nparts; ++p) v += bad(p);
    violations[i] = v;
  }
  return HGP_REF_OK;
}

// f4: the landing point: among the prefixes k = 1..M whose last move leaves no
// violated constraint, the largest cumulative in-sequence gain (the shortest prefix on ties);
// nothing is applied unless that gain is > 0.
int hgp_ref_best_prefix(const int64_t *gain_seq, const uint32_t *violations, uint32_t M, uint32_t *k, int64_t *best) {
  if (!k || !best || (M && (!gain_seq || !violations))) return hgp_ref_set_error(HGP_REF_E_ARG, "null argument");
  int64_t cum = 0, bv = 0;
  uint32_t bk = 0;
  for (uint32_t i = 0; i < M; ++i) {
    cum += gain_seq[i];
    if (violations[i] == 0 && cum > bv) { bv = cum; bk = i + 1; }
  }
  *k = bk;
  *best = bv;
  return HGP_REF_OK;
}

}  // extern "C"
