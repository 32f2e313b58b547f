"""Oracle vs brute force: all-pairs scoring via incidence-matrix products, explicit
set unions, exhaustive matching enumeration, batch independence."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests import _pins

NONE = ref.NONE


def small_graphs():
    yield "tiny-60", hgpgen.tiny(11, num_nodes=60, num_edges=120, size_binom=6, in_cap=12, wmax_e=8, wmax_n=3), 6, 14
    yield "tiny-200", hgpgen.tiny(12, num_nodes=200, num_edges=500, in_cap=20, wmax_e=5), 16, 24
    yield "C1-seed1", hgpgen.tiny(1), 16, 32
    yield "snn-small", hgpgen.snn(3, layers=3, rows=8, cols=8, fanout=12, window=5, rewire=0.1), 8, 40
    yield "vlsi-small", hgpgen.vlsi(4, 400, 400, dmax=40, in_cap=30), 8, 40


@pytest.mark.parametrize("name,hg,omega,delta", list(small_graphs()), ids=lambda x: x if isinstance(x, str) else "")
@pytest.mark.parametrize("norm,noise_cap", [(0, 0), (0, 1 << 22), (1, 0)])
def test_a1_a2_a3_against_matrix_products(name, hg, omega, delta, norm, noise_cap):
    g = ref.build_csr_hg(hg)
    edges = _pins.edges_of(hg.edge_off, hg.edge_nsrc, hg.pins)
    # a1: canonical pins (sorted src / dst blocks, same sets) and brute-force incidence.
    for e, (S, D) in enumerate(_pins.edges_of(g.edge_off, g.edge_nsrc, g.pins)):
        lo, s, hi = int(g.edge_off[e]), int(g.edge_off[e]) + int(g.edge_nsrc[e]), int(g.edge_off[e + 1])
        assert (S, D) == edges[e]
        assert list(g.pins[lo:s]) == sorted(S) and list(g.pins[s:hi]) == sorted(D)
    ins, outs = _pins.incidence_bruteforce(hg.num_nodes, edges)
    for n in range(hg.num_nodes):
        lo, nin, hi = int(g.inc_off[n]), int(g.inc_nin[n]), int(g.inc_off[n + 1])
        assert list(g.inc[lo:lo + nin]) == ins[n] and list(g.inc[lo + nin:hi]) == outs[n]
    assert int(g.inc_off[-1]) == hg.num_pins                      # sum |I(n)| = sum |e|
    # a2 + a3 by matrix products
    bf = _pins.score_bruteforce(hg.num_nodes, g.edge_off, g.edge_nsrc, g.pins, g.edge_w, g.edge_mu, g.node_w,
                                omega, delta, 4, norm=norm, seed=77, cap=noise_cap)
    nb = ref.unique_neighbors(g)
    for n in range(hg.num_nodes):
        assert list(nb.segment(n)) == list(np.nonzero(bf["adj"][n])[0])
    cand = ref.score_pairs(g, nb, ref.params(omega, delta, 4, norm=norm, noise_seed=77, noise_cap=noise_cap))
    for n in range(hg.num_nodes):
        got = [(int(c["id"]), int(c["score"])) for c in cand[n] if c["id"] != NONE]
        assert got == bf["cand"][n], n
    flagged = {(n, int(v) & 0x7FFFFFFF) for n in range(hg.num_nodes) for v in nb.segment(n) if v & ref.PURGE}
    assert flagged == bf["flagged"]
    # flags are symmetric because validity is
    assert all((m, n) in flagged for (n, m) in flagged)


def test_inline_intersection_equals_explicit_union():
    """|in(n) ∪ in(m)| = |in(n)| + |in(m)| - inter(n,m) against explicit set unions."""
    hg = hgpgen.tiny(5, num_nodes=150, num_edges=400, in_cap=6)
    g = ref.build_csr_hg(hg)
    edges = _pins.edges_of(g.edge_off, g.edge_nsrc, g.pins)
    ins, _ = _pins.incidence_bruteforce(hg.num_nodes, edges)
    bf = _pins.score_bruteforce(hg.num_nodes, g.edge_off, g.edge_nsrc, g.pins, g.edge_w, g.edge_mu, g.node_w,
                                10 ** 9, 10 ** 9, 4)
    for n in range(hg.num_nodes):
        for m in np.nonzero(bf["adj"][n])[0]:
            m = int(m)
            union = len(set(ins[n]) | set(ins[m]))
            assert union == int(g.in_mu[n]) + int(g.in_mu[m]) - int(bf["inter"][n, m])
    # and the oracle's validity decisions use exactly that count: Delta = the union size boundary
    nb = ref.unique_neighbors(g)
    delta = 8
    ref.score_pairs(g, nb, ref.params(10 ** 9, delta, 4))
    for n in range(hg.num_nodes):
        for v in nb.segment(n):
            m = int(v) & 0x7FFFFFFF
            assert bool(v & ref.PURGE) == (len(set(ins[n]) | set(ins[m])) > delta)


@pytest.mark.parametrize("batch", [1, 2, 7, 64])
def test_batch_independence(batch):
    """Results must not depend on the neighbour batch size."""
    hg = hgpgen.tiny(21, num_nodes=300, num_edges=800, in_cap=16)
    g = ref.build_csr_hg(hg)
    nb0, nb1 = ref.unique_neighbors(g), ref.unique_neighbors(g)
    p0 = ref.params(16, 20, 4, noise_seed=3, noise_cap=1 << 20)
    p1 = ref.params(16, 20, 4, noise_seed=3, noise_cap=1 << 20, batch=batch)
    c0, c1 = ref.score_pairs(g, nb0, p0), ref.score_pairs(g, nb1, p1)
    assert np.array_equal(c0, c1) and np.array_equal(nb0.nbr, nb1.nbr)


def test_noise_is_symmetric_and_capped():
    hg = hgpgen.tiny(8, num_nodes=80, num_edges=200)
    g = ref.build_csr_hg(hg)
    cap = (1 << 23) + 17
    bf0 = _pins.score_bruteforce(hg.num_nodes, g.edge_off, g.edge_nsrc, g.pins, g.edge_w, g.edge_mu, g.node_w,
                                 10 ** 9, 10 ** 9, 16)
    nb = ref.unique_neighbors(g)
    cand = ref.score_pairs(g, nb, ref.params(10 ** 9, 10 ** 9, 16, noise_seed=5, noise_cap=cap))
    sc = {}
    for n in range(hg.num_nodes):
        for c in cand[n]:
            if c["id"] != NONE:
                sc[(n, int(c["id"]))] = int(c["score"])
    assert sc
    for (n, m), s in sc.items():
        assert 0 <= s - int(bf0["eta"][n, m]) <= cap
        if (m, n) in sc:
            assert sc[(m, n)] == s


def _random_cand(rng, N, pi, p_edge=0.3, levels=4):
    """Random symmetric eta with many ties + random symmetric validity -> top-pi cand arrays."""
    eta = np.zeros((N, N), dtype=np.int64)
    ok = np.zeros((N, N), dtype=bool)
    for a in range(N):
        for b in range(a + 1, N):
            if rng.random() < p_edge:
                eta[a, b] = eta[b, a] = int(rng.integers(1, levels + 1))
                ok[a, b] = ok[b, a] = rng.random() < 0.8
    cand = np.zeros((N, pi), dtype=ref.CAND_DTYPE)
    cand["id"] = NONE
    for n in range(N):
        vals = sorted(((int(eta[n, m]), m) for m in range(N) if eta[n, m] > 0 and ok[n, m]), key=lambda t: (-t[0], -t[1]))
        for i, (s, m) in enumerate(vals[:pi]):
            cand[n, i] = (m, 0, s)
    return cand


def _rounds(cand, pi):
    """Per-round matches: rounds are sequential, so the first k rounds of a Pi-round run are
    exactly a k-round run on cand[:, :k]. Yields (t, s, new_pairs, value, pairs_count)."""
    N = cand.shape[0]
    prev = np.full(N, NONE, dtype=np.uint32)
    matched = [False] * N
    for i in range(pi):
        mk, per, val = ref.match(np.ascontiguousarray(cand[:, :i + 1]), i + 1)
        t, s = _pins.round_graph(cand, i, matched)
        new = [(n, int(mk[n])) for n in range(N) if prev[n] == NONE and mk[n] != NONE and n < mk[n]]
        yield t, s, new, int(val[i]), int(per[i])
        for a, b in new:
            matched[a] = matched[b] = True
        assert all(prev[n] == NONE or prev[n] == mk[n] for n in range(N))   # earlier rounds are final
        prev = mk


def test_matching_against_exhaustive_enumeration():
    """Per round: two-cycle pseudo-forest, DP optimum = exhaustive maximum, and the oracle's
    new pairs realise it (acceptance #1)."""
    rng = np.random.default_rng(2024)
    checked = 0
    for trial in range(500):
        N = int(rng.integers(2, 13))
        pi = int(rng.integers(1, 5))
        cand = _random_cand(rng, N, pi)
        for t, s, new, val, npairs in _rounds(cand, pi):
            assert _pins.has_only_two_cycles(t)
            ew = {(min(n, t[n]), max(n, t[n])): s[n] for n in range(N) if t[n] != NONE}
            best = _pins.max_matching_bruteforce(range(N), ew)
            assert best == val
            assert all(p in ew for p in new)                 # matches follow proposal edges
            assert sum(ew[p] for p in new) == best and len(new) == npairs
            checked += 1
        m, _, _ = ref.match(cand, pi)
        for n in range(N):
            if m[n] != NONE:
                assert m[m[n]] == n
    assert checked > 500


def test_matching_rounds_on_c1_components():
    """On C1, every round's proposal graph is a two-cycle pseudo-forest and each small
    component's DP result equals exhaustive search."""
    hg = hgpgen.tiny(1)
    g = ref.build_csr_hg(hg)
    nb = ref.unique_neighbors(g)
    cand = ref.score_pairs(g, nb, ref.params(16, 32, 4, noise_seed=9, noise_cap=1 << 22))
    small = 0
    for i, (t, s, new, val, npairs) in enumerate(_rounds(cand, 4)):
        assert _pins.has_only_two_cycles(t)
        if i == 0:   # score(target(n)) >= score(n) along every round-1 proposal edge
            assert all(s[t[n]] >= s[n] for n in range(g.N) if t[n] != NONE)
        newset = set(new)
        total = 0
        for comp in _pins.proposal_components(t):
            ew = {(min(n, t[n]), max(n, t[n])): s[n] for n in comp if t[n] != NONE}
            got = sum(ew[p] for p in ew if p in newset)
            total += got
            if len(comp) <= 18 and ew:
                assert got == _pins.max_matching_bruteforce(comp, ew)
                small += 1
        assert total == val and len(new) == npairs
    assert small > 50
