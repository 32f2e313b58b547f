"""Oracle contraction vs the level's invariants I1-I6, over several
levels so that merged parallel edges (mu > 1) and propagated purge flags are exercised."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests import _pins

NONE = ref.NONE


def check_level(g, nb_after_score, r, omega, delta, rng):
    """I1-I6 for one contraction g -> r['coarse'] with gamma r['gamma']."""
    gamma, cg, cnb, m = r["gamma"], r["coarse"], r["coarse_nb"], r["match"]
    N, Nc = g.N, cg.N
    edges = _pins.edges_of(g.edge_off, g.edge_nsrc, g.pins)
    cedges = _pins.edges_of(cg.edge_off, cg.edge_nsrc, cg.pins)
    # gamma: clusters of <= 2 nodes, coarse ids by ascending min member (reading #11)
    assert Nc == N - sum(1 for n in range(N) if m[n] != NONE) // 2
    firsts = [min(n for n in range(N) if gamma[n] == c) for c in range(Nc)]
    assert firsts == sorted(firsts)
    # I1 total size conserved
    assert int(cg.node_w.astype(np.int64).sum()) == int(g.node_w.astype(np.int64).sum())
    # I2 every coarse node respects Omega and Delta
    assert all(int(x) <= omega for x in cg.node_w)
    if delta != ref.UNBOUNDED:
        assert all(int(x) <= delta for x in cg.in_mu)
    # I3 pin projection: each kept fine edge's class key maps to a coarse edge with summed weights
    keyed = {}
    dropped_w = 0
    for e, (S, D) in enumerate(edges):
        Dp = {int(gamma[x]) for x in D}
        Sp = {int(gamma[x]) for x in S} - Dp
        if not Dp and len(Sp) <= 1:
            dropped_w += int(g.edge_w[e])
            continue
        k = (frozenset(Sp), frozenset(Dp))
        w, mu, rep = keyed.get(k, (0, 0, e))
        keyed[k] = (w + int(g.edge_w[e]), mu + int(g.edge_mu[e]), min(rep, e))
    got = {(frozenset(S), frozenset(D)): (int(cg.edge_w[e]), int(cg.edge_mu[e])) for e, (S, D) in enumerate(cedges)}
    assert len(got) == cg.E                                   # no two coarse edges are parallel
    assert got == {k: v[:2] for k, v in keyed.items()}
    reps = sorted(v[2] for v in keyed.values())               # coarse order = ascending representative
    assert [keyed[(frozenset(S), frozenset(D))][2] for (S, D) in cedges] == reps
    # I4 connectivity, cut-net and Delta-counts of random coarse partitions equal their projections
    for trial in range(6):
        k = int(rng.integers(1, max(2, Nc // 3) + 1)) if trial else Nc
        rho_c = rng.integers(0, k, size=Nc) if trial else np.arange(Nc)
        rho_f = rho_c[gamma]
        assert _pins.connectivity(cedges, cg.edge_w, rho_c) == _pins.connectivity(edges, g.edge_w, rho_f)
        assert _pins.cut_net(cedges, cg.edge_w, rho_c) == _pins.cut_net(edges, g.edge_w, rho_f)
        assert _pins.inbound_counts(cedges, cg.edge_mu, rho_c, k) == _pins.inbound_counts(edges, g.edge_mu, rho_f, k)
    # in_mu' = distinct original inbound edges of the cluster
    assert list(cg.in_mu) == _pins.inbound_counts(edges, g.edge_mu, gamma, Nc)
    # I5 duality: Score(gamma) + Conn(gamma) = sum omega (|e| - 1)
    total = sum(int(g.edge_w[e]) * (len(S | D) - 1) for e, (S, D) in enumerate(edges))
    assert _pins.coarsening_score(edges, g.edge_w, gamma) + _pins.connectivity(edges, g.edge_w, gamma) == total
    # I6 N' = true coarse neighbourhood minus OR-propagated flags, symmetric
    true_nb = [set() for _ in range(Nc)]
    for (S, D) in cedges:
        pins = S | D
        for a in pins:
            true_nb[a] |= pins - {a}
    flagged = [set() for _ in range(Nc)]
    for n in range(N):
        for v in nb_after_score.segment(n):
            if int(v) & ref.PURGE:
                flagged[int(gamma[n])].add(int(gamma[int(v) & 0x7FFFFFFF]))
    # fine-level view: which fine neighbours were already gone before this level's scoring
    fine_true = [set() for _ in range(N)]
    for (S, D) in edges:
        for a in S | D:
            fine_true[a] |= (S | D) - {a}
    for c in range(Nc):
        seg = [int(x) for x in cnb.segment(c)]
        assert seg == sorted(seg) and all(x & ref.PURGE == 0 for x in seg)
        # sound: every surviving entry is a true coarse neighbour and none is flagged
        assert set(seg) <= true_nb[c] and not (set(seg) & flagged[c])
        members = [n for n in range(N) if gamma[n] == c]
        complete = all(set(int(v) & 0x7FFFFFFF for v in nb_after_score.segment(a)) == fine_true[a] for a in members)
        if complete:   # no earlier purge touched these members: N' is exactly the true set minus flags
            assert set(seg) == true_nb[c] - flagged[c]
    for c in range(Nc):
        for x in cnb.segment(c):
            assert c in set(int(y) for y in cnb.segment(int(x)))


CASES = [
    ("C1", lambda: hgpgen.tiny(1), 16, 32),
    ("C1-w3", lambda: hgpgen.tiny(2, wmax_n=3), 16, 32),
    ("dense-small", lambda: hgpgen.tiny(3, num_nodes=120, num_edges=600, size_binom=4, in_cap=40), 8, 48),
    ("snn-small", lambda: hgpgen.snn(5, layers=4, rows=10, cols=10, fanout=15, window=5, rewire=0.1), 16, 64),
    ("vlsi-small", lambda: hgpgen.vlsi(6, 500, 500, dmax=60, in_cap=40), 16, 64),
    ("kway", lambda: hgpgen.vlsi(7, 300, 300, dmax=30, in_cap=1000), 155, ref.UNBOUNDED),
]


@pytest.mark.parametrize("name,make,omega,delta", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("cap", [0, 1 << 22])
def test_invariants_over_levels(name, make, omega, delta, cap):
    hg = make()
    g = ref.build_csr_hg(hg)
    nb = ref.unique_neighbors(g)
    rng = np.random.default_rng(99)
    for level in range(4):
        p = ref.params(omega, delta, 4, noise_seed=level, noise_cap=cap)
        nb_before = nb.copy()
        r = ref.coarsen_level(g, nb, p)
        # flags only ever get added by scoring
        assert np.array_equal(nb.nbr & 0x7FFFFFFF, nb_before.nbr & 0x7FFFFFFF)
        check_level(g, nb, r, omega, delta, rng)
        g, nb = r["coarse"], r["coarse_nb"]
        if g.N < 4:
            break


def test_parallel_edges_merge_with_multiplicity():
    """e1: src{0} dst{2}, e2: src{1} dst{2}; matching 0-1 makes them parallel (S'={c01}, D'={c2}):
    one coarse edge, omega' = 3 + 4, mu' = 2, and |in(c2)| still counts both originals."""
    g = ref.build_csr(3, [0, 2, 4], [1, 1], [0, 2, 1, 2], [3, 4], [1, 1, 1])
    nb = ref.unique_neighbors(g)
    gamma, cg, cnb = ref.contract(g, nb, np.array([1, 0, NONE], dtype=np.uint32))
    assert list(gamma) == [0, 0, 1] and cg.E == 1
    assert list(cg.pins) == [0, 1] and list(cg.edge_nsrc) == [1]
    assert list(cg.edge_w) == [7] and list(cg.edge_mu) == [2] and list(cg.in_mu) == [0, 2]


def test_coarse_level_neighbors_equal_recomputed_minus_flags():
    """I6 exactly: with no flags set, N' equals hgp_ref_unique_neighbors on G'."""
    hg = hgpgen.tiny(4)
    g = ref.build_csr_hg(hg)
    nb = ref.unique_neighbors(g)
    r = ref.coarsen_level(g, nb, ref.params(10 ** 6, 10 ** 6, 4))   # unconstrained: no flags
    assert not (nb.nbr & ref.PURGE).any()
    again = ref.unique_neighbors(r["coarse"])
    assert np.array_equal(again.off, r["coarse_nb"].off) and np.array_equal(again.nbr, r["coarse_nb"].nbr)


def test_matched_fraction_grows_with_pi():
    """Direction of the Pi ablation (acceptance #10): Pi=4 matches more nodes than Pi=1."""
    hg = hgpgen.tiny(9)
    g = ref.build_csr_hg(hg)
    frac = {}
    for pi in (1, 4):
        nb = ref.unique_neighbors(g)
        r = ref.coarsen_level(g, nb, ref.params(16, 32, pi, noise_seed=1, noise_cap=1 << 22))
        frac[pi] = float((r["match"] != NONE).mean())
    assert frac[4] > frac[1]
