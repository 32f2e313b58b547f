"""Oracle vs the paper's / SPEC's worked examples (tests/golden/h_ex.json, each entry cited)."""
import json
import os

import numpy as np
import pytest

from oracle import ref
from tests import _pins

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "h_ex.json")))
G = GOLD["graph"]


def hex_csr():
    return ref.build_csr(G["num_nodes"], G["edge_off"], G["edge_nsrc"], G["pins"], G["edge_w"], G["node_w"])


def test_splitmix64_known_answers():
    # SplitMix64 reference generator (Steele, Lea, Flood 2014; Vigna's splitmix64.c):
    # first output from state 0 is 0xE220A8397B1DCDAF.
    assert _pins.splitmix64(0) == 0xE220A8397B1DCDAF


def test_metrics_helpers_against_spec():
    m = GOLD["metrics"]
    edges = _pins.edges_of(np.array(G["edge_off"]), G["edge_nsrc"], G["pins"])
    assert _pins.connectivity(edges, G["edge_w"], m["rho"]) == m["connectivity"]
    assert _pins.connectivity(edges, G["edge_w"], [0, 1, 2, 3]) == m["connectivity_singletons"]
    assert _pins.cut_net(edges, G["edge_w"], m["rho"]) == m["cut_net"]
    assert _pins.coarsening_score(edges, G["edge_w"], m["rho"]) == m["score"]
    assert m["score"] + m["connectivity"] == m["duality_total"]


def test_incidence_and_neighbors():
    g = hex_csr()
    for n in range(4):
        lo, hi = int(g.inc_off[n]), int(g.inc_off[n + 1])
        nin = int(g.inc_nin[n])
        assert list(g.inc[lo:lo + nin]) == GOLD["incidence"]["in"][n]
        assert list(g.inc[lo + nin:hi]) == GOLD["incidence"]["out"][n]
        assert g.in_mu[n] == len(GOLD["incidence"]["in"][n])
    nb = ref.unique_neighbors(g)
    assert [list(nb.segment(n)) for n in range(4)] == GOLD["neighbors"]["nbr"]


def test_eta_fixed_point():
    g = hex_csr()
    nb = ref.unique_neighbors(g)
    cand = ref.score_pairs(g, nb, ref.params(100, 100, 4))
    got = {}
    for n in range(4):
        for c in cand[n]:
            if c["id"] != ref.NONE:
                got[(n, int(c["id"]))] = int(c["score"])
    for n, m, v in GOLD["eta"]["pairs"]:
        assert got[(n, m)] == v


@pytest.mark.parametrize("case", ["case_A", "case_B"])
def test_appendix_a_cases(case):
    c = GOLD[case]
    g = hex_csr()
    nb = ref.unique_neighbors(g)
    r = ref.coarsen_level(g, nb, ref.params(c["omega"], c["delta"], c["pi"]))
    cand = [[[int(x["id"]), int(x["score"])] for x in row if x["id"] != ref.NONE] for row in r["cand"]]
    assert cand == c["cand"]
    flagged = sorted([n, int(v) & 0x7FFFFFFF] for n in range(4) for v in nb.segment(n) if v & ref.PURGE)
    assert flagged == sorted(c["flagged"])
    assert [None if x == ref.NONE else int(x) for x in r["match"]] == c["match"]
    assert list(r["gamma"]) == c["gamma"]
    cg, cnb = r["coarse"], r["coarse_nb"]
    assert [list(cnb.segment(x)) for x in range(cg.N)] == c["coarse_nbr"]
    if "coarse_edges" in c:
        assert list(cg.node_w) == c["coarse_node_w"]
        ed = []
        for e in range(cg.E):
            lo, hi = int(cg.edge_off[e]), int(cg.edge_off[e + 1])
            s = lo + int(cg.edge_nsrc[e])
            ed.append([list(cg.pins[lo:s]), list(cg.pins[s:hi]), int(cg.edge_w[e]), int(cg.edge_mu[e])])
        assert ed == c["coarse_edges"]
        assert list(cg.in_mu) == c["coarse_in_mu"]


def test_infeasible_node_is_named():
    c = GOLD["infeasible"]
    g = hex_csr()
    nb = ref.unique_neighbors(g)
    with pytest.raises(ref.OracleError) as ei:
        ref.score_pairs(g, nb, ref.params(c["omega"], c["delta"], 4))
    assert ei.value.code == -3 and f"node {c['node']}" in ei.value.msg


def _cand_array(rows, pi):
    cand = np.zeros((len(rows), pi), dtype=ref.CAND_DTYPE)
    cand["id"] = ref.NONE
    for n, row in enumerate(rows):
        for i, (m, s) in enumerate(row):
            cand[n, i] = (m, 0, s)
    return cand


def test_dp_example():
    c = GOLD["dp_example"]
    m, per, val = ref.match(_cand_array(c["cand"], 1))
    assert list(m) == c["match"] and int(val[0]) == c["total"]


def test_star_two_rounds():
    c = GOLD["star_two_rounds"]
    m, per, val = ref.match(_cand_array(c["cand"], 2))
    assert list(m) == c["match"] and list(per) == c["matched_per_round"]


def test_gamma_compaction():
    c = GOLD["gamma_compaction"]
    # 4 isolated nodes: neighbours are empty, only gamma matters.
    g = ref.build_csr(4, [0], [], [], [], [1, 1, 1, 1])
    nb = ref.unique_neighbors(g)
    match = np.array([ref.NONE if x is None else x for x in c["match"]], dtype=np.uint32)
    gamma, cg, _ = ref.contract(g, nb, match)
    assert list(gamma) == c["gamma"] and list(cg.node_w) == [2, 1, 1]


@pytest.mark.parametrize("bad,code,idx", [
    (dict(edge_off=[0, 2, 2], edge_nsrc=[1, 0], pins=[0, 1]), -2, "edge 1"),            # empty edge
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 1], pins=[0, 1, 2, 2]), -2, "edge 1"),      # duplicate pin
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 1], pins=[0, 1, 1, 1]), -2, "edge 1"),      # src ∩ dst
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 3], pins=[0, 1, 1, 2]), -2, "edge 1"),      # nsrc > |e|
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 1], pins=[0, 1, 1, 9]), -2, "edge 1"),      # pin >= N
])
def test_malformed_inputs(bad, code, idx):
    E = len(bad["edge_nsrc"])
    with pytest.raises(ref.OracleError) as ei:
        ref.build_csr(4, bad["edge_off"], bad["edge_nsrc"], bad["pins"], [1] * E, [1] * 4)
    assert ei.value.code == code and idx in ei.value.msg


def test_zero_weights_rejected():
    with pytest.raises(ref.OracleError) as ei:
        ref.build_csr(3, [0, 2], [1], [0, 1], [0], [1, 1, 1])
    assert ei.value.code == -2 and "edge 0" in ei.value.msg
    with pytest.raises(ref.OracleError) as ei:
        ref.build_csr(3, [0, 2], [1], [0, 1], [1], [1, 0, 1])
    assert ei.value.code == -2 and "node 1" in ei.value.msg
