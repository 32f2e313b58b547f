"""Oracle a3 pinned at COARSE levels, where merged parallel edges carry multiplicity mu > 1.

Level 0 has mu = 1 everywhere, so the level-0 brute-force pins cannot tell
``inter += mu(e)`` (reading #12) from ``inter += 1``.  Here the oracle runs up to 4
levels deep and, at every coarse level:

* cand and purge flags equal the matrix-product brute force fed the coarse edge_mu
  (``_pins.score_bruteforce`` with ``live`` = the unflagged coarse neighbours);
* every validity decision equals the paper's own definition evaluated on the ORIGINAL level-0
  hypergraph: |{e0 : dst(e0) meets rho^-1(n) ∪ rho^-1(m)}| <= Delta and size <= Omega
  (P:305-311 — the distinct inbound hyperedges of the merged cluster), with rho the composed
  gammas.  No mu, no coarse edge list: an explicit set union of original edge ids.

The instances are chosen so that the pins are *sensitive*: some coarse pair's validity flips if
mu is replaced by 1 (asserted), so a dropped multiplicity fails this file.
"""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests import _pins

NONE = ref.NONE


def _live(cnb, N):
    return [set(int(v) for v in cnb.segment(n) if not (int(v) & ref.PURGE)) for n in range(N)]


def _orig_inbound_sets(g0):
    """in0[n] = set of original edge ids with n in dst."""
    edges = _pins.edges_of(g0.edge_off, g0.edge_nsrc, g0.pins)
    ins = [set() for _ in range(g0.N)]
    for e, (_, D) in enumerate(edges):
        for x in D:
            ins[x].add(e)
    return ins


def _mu1_inter(g, n, m):
    """inter(n, m) as a3 would compute it with mu dropped: shared coarse in-edges counted once."""
    lo_n, lo_m = int(g.inc_off[n]), int(g.inc_off[m])
    a = set(int(x) for x in g.inc[lo_n:lo_n + int(g.inc_nin[n])])
    b = set(int(x) for x in g.inc[lo_m:lo_m + int(g.inc_nin[m])])
    return len(a & b)


CASES = [
    # name, generator, Omega, Delta, levels, must_be_mu_sensitive. Small edges so that contraction
    # makes parallel edges; the SNN windows make merged all-destination edges shared by neighbours,
    # so with Delta near the clusters' in-degrees some validity decisions hinge on mu.
    ("tiny-2to3", lambda: hgpgen.tiny(31, num_nodes=120, num_edges=420, size_base=2, size_binom=1, in_cap=14,
                                      wmax_e=4), 8, 24, 4, False),
    ("vlsi-small", lambda: hgpgen.vlsi(33, 300, 300, dmax=12, in_cap=20), 16, 24, 4, False),
    ("snn-d16", lambda: hgpgen.snn(33, layers=3, rows=6, cols=6, fanout=8, window=3, rewire=0.0), 8, 16, 4, True),
    ("snn-d20", lambda: hgpgen.snn(33, layers=3, rows=6, cols=6, fanout=8, window=3, rewire=0.0), 16, 20, 4, True),
    ("snn-d24", lambda: hgpgen.snn(33, layers=3, rows=6, cols=6, fanout=8, window=3, rewire=0.0), 16, 24, 4, True),
]


@pytest.mark.parametrize("name,make,omega,delta,levels,must", CASES, ids=[c[0] for c in CASES])
def test_coarse_level_a3_against_bruteforce_and_original_unions(name, make, omega, delta, levels, must):
    hg = make()
    g0 = ref.build_csr_hg(hg)
    in0 = _orig_inbound_sets(g0)
    g, nb = g0, ref.unique_neighbors(g0)
    rho = np.arange(g0.N, dtype=np.uint32)
    merged_levels = 0
    sensitive = 0
    checked_pairs = 0
    for lvl in range(levels):
        p = ref.params(omega, delta, 4, noise_seed=5 + lvl, noise_cap=1 << 21)
        if lvl > 0:
            # ---- the pins at this coarse level (flags of this level are set by score_pairs)
            live = _live(nb, g.N)
            bf = _pins.score_bruteforce(g.N, g.edge_off, g.edge_nsrc, g.pins, g.edge_w, g.edge_mu, g.node_w,
                                        omega, delta, 4, seed=5 + lvl, cap=1 << 21, live=live)
            nb_s = nb.copy()
            cand = ref.score_pairs(g, nb_s, p)
            for n in range(g.N):
                got = [(int(c["id"]), int(c["score"])) for c in cand[n] if c["id"] != NONE]
                assert got == bf["cand"][n], (lvl, n)
            flagged = {(n, int(v) & 0x7FFFFFFF) for n in range(g.N) for v in nb_s.segment(n) if int(v) & ref.PURGE}
            assert flagged == bf["flagged"], lvl
            # the paper's definition on the ORIGINAL hypergraph, cluster by cluster
            members = [[] for _ in range(g.N)]
            for x in range(g0.N):
                members[int(rho[x])].append(x)
            cin = [set().union(*(in0[x] for x in members[c])) if members[c] else set() for c in range(g.N)]
            csize = [sum(int(g0.node_w[x]) for x in members[c]) for c in range(g.N)]
            assert csize == [int(x) for x in g.node_w]
            assert [len(s) for s in cin] == [int(x) for x in g.in_mu]           # in_mu' = |in(cluster)|
            for n in range(g.N):
                for m in live[n]:
                    uni = len(cin[n] | cin[m])
                    valid = csize[n] + csize[m] <= omega and uni <= delta
                    assert valid == ((n, m) not in flagged), (lvl, n, m)
                    # the union a3 reads off its inline counter equals the original-edge union
                    assert int(g.in_mu[n]) + int(g.in_mu[m]) - int(bf["inter"][n, m]) == uni
                    if csize[n] + csize[m] <= omega and (uni <= delta) != (
                            int(g.in_mu[n]) + int(g.in_mu[m]) - _mu1_inter(g, n, m) <= delta):
                        sensitive += 1
                    checked_pairs += 1
        if int(g.edge_mu.max(initial=0)) > 1:
            merged_levels += 1
        r = ref.coarsen_level(g, nb, p)
        rho = r["gamma"][rho]
        g, nb = r["coarse"], r["coarse_nb"]
        if g.N < 4:
            break
    assert merged_levels >= 1, "no merged parallel edge (mu > 1) was scored: the pin is vacuous"
    assert checked_pairs > 50
    print(name, "pairs", checked_pairs, "mu-sensitive", sensitive)
    assert sensitive >= 1 or not must, "no pair whose validity depends on mu: the pin is not sensitive"
