"""Oracle f2 — deterministic best-effort pairing of the nodes left without any candidate
(DESIGN reading #22), pinned independently of its own loops:
  * a hand-derived example (targets, the DP's choice of two child pairs over the mutual pair);
  * targets = the paper's formulation (sort by size, search down from the slack for the first
    valid node, ties by id), written as a sort + scan instead of the oracle's max loop;
  * the proposal graph has only 2-cycles (symmetric score, consistent ties);
  * the DP optimum of the extra round equals exhaustive enumeration over the proposal edges;
  * a level with f2 keeps every coarse node within Omega and Delta and matches at least as many
    pairs as without it."""
import itertools

import numpy as np
import pytest

import hgpgen
from oracle import ref

NONE = ref.NONE


def _cand_none(n):
    c = np.zeros((n, 1), dtype=ref.CAND_DTYPE)
    c["id"] = NONE
    return c


def test_hand_example():
    # four nodes without neighbours, sizes 1,2,3,1, Omega = 4, Delta unbounded
    w = np.array([1, 2, 3, 1], dtype=np.uint32)
    mu = np.zeros(4, dtype=np.uint32)
    t = ref.leftover_targets(_cand_none(4), w, mu, 4, ref.UNBOUNDED)
    assert [int(x) for x in t["id"][:, 0]] == [2, 3, 3, 2]
    assert [int(x) for x in t["score"][:, 0]] == [4, 3, 4, 4]
    m, added = ref.leftover_pairs(_cand_none(4), w, mu, 4, ref.UNBOUNDED, np.full(4, NONE, dtype=np.uint32))
    # root pair 2<->3 is worth 4; its children 0->2 (4) and 1->3 (3) together are worth 7
    assert list(m) == [2, 3, 0, 1] and added == 2


def _paper_targets(cand, w, mu, omega, delta):
    """P:674-677 as written: L sorted by size; per node, binary search for the size slack, then
    walk down to the first valid node (ids break ties: the larger id is met first)."""
    N = cand.shape[0]
    L = [n for n in range(N) if int(cand[n][0]["id"]) == NONE]
    order = sorted(L, key=lambda n: (int(w[n]), n))
    sizes = [int(w[n]) for n in order]
    out = {}
    for n in L:
        slack = omega - int(w[n])
        j = int(np.searchsorted(np.array(sizes, dtype=np.int64), slack, side="right")) - 1
        while j >= 0:
            m = order[j]
            if m != n and (delta == ref.UNBOUNDED or int(mu[n]) + int(mu[m]) <= delta):
                out[n] = m
                break
            j -= 1
    return out


@pytest.mark.parametrize("seed", range(40))
def test_targets_two_cycles_and_dp_optimum(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 11))
    w = rng.integers(1, 5, size=N).astype(np.uint32)
    mu = rng.integers(0, 4, size=N).astype(np.uint32)
    omega, delta = int(rng.integers(2, 8)), (ref.UNBOUNDED if seed % 3 == 0 else int(rng.integers(0, 6)))
    cand = _cand_none(N)
    # some nodes have a regular candidate: they are not leftovers
    for n in range(N):
        if rng.random() < 0.25:
            cand[n, 0] = ((n + 1) % N, 0, 1)
    t = ref.leftover_targets(cand, w, mu, omega, delta)
    tgt = {n: int(t[n, 0]["id"]) for n in range(N) if int(t[n, 0]["id"]) != NONE}
    assert tgt == _paper_targets(cand, w, mu, omega, delta)
    # scores and validity
    for n, m in tgt.items():
        assert int(t[n, 0]["score"]) == int(w[n]) + int(w[m]) and int(w[n]) + int(w[m]) <= omega
        assert delta == ref.UNBOUNDED or int(mu[n]) + int(mu[m]) <= delta
    # only 2-cycles
    for n in tgt:
        seen, x = [], n
        while x in tgt and x not in seen:
            seen.append(x)
            x = tgt[x]
        if x in seen:
            assert len(seen) - seen.index(x) == 2
    # DP optimum == best matching that uses proposal edges only
    m, added = ref.leftover_pairs(cand, w, mu, omega, delta, np.full(N, NONE, dtype=np.uint32))
    edges = {(min(a, b), max(a, b)): int(w[a]) + int(w[b]) for a, b in tgt.items()}
    best = 0
    E = list(edges.items())
    for r in range(len(E) + 1):
        for sub in itertools.combinations(E, r):
            nodes = [x for (a, b), _ in sub for x in (a, b)]
            if len(nodes) == len(set(nodes)):
                best = max(best, sum(s for _, s in sub))
    got = sum(int(w[n]) + int(w[int(m[n])]) for n in range(N) if m[n] != NONE and n < m[n])
    assert got == best
    for n in range(N):
        if m[n] != NONE:
            assert m[int(m[n])] == n and (int(m[n]), n) in [(b, a) for a, b in tgt.items()] + list(tgt.items())


@pytest.mark.parametrize("make,omega,delta", [
    (lambda: hgpgen.tiny(5, num_nodes=300, num_edges=200, size_binom=4), 4, 8),
    (lambda: hgpgen.vlsi(9, 400, 300, dmax=20, in_cap=12), 6, 14),
])
def test_level_with_leftover_respects_constraints(make, omega, delta):
    hg = make()
    g = ref.build_csr_hg(hg)
    a = ref.coarsen_level(g, ref.unique_neighbors(g), ref.params(omega, delta, 4))
    b = ref.coarsen_level(g, ref.unique_neighbors(g), ref.params(omega, delta, 4), leftover=True)
    assert (b["match"] != NONE).sum() >= (a["match"] != NONE).sum()
    cg = b["coarse"]
    assert int(cg.node_w.max()) <= omega and int(cg.in_mu.max()) <= delta
    assert int(cg.node_w.astype(np.int64).sum()) == int(g.node_w.astype(np.int64).sum())
