"""Oracle multi-level driver against what the paper fixes for the
whole hierarchy, independently of the per-level code:
  * the stop rule (reading #20) holds at the last level and at no earlier one;
  * the composed map rho = gamma^L o ... o gamma^1 conserves size and every coarsest
    node respects Omega and — counted on the ORIGINAL level-0 edges — Delta (Eq.6), which
    pins the multiplicity mu carried through every merge of parallel edges (reading #12);
  * connectivity / cut-net of any partition of the coarsest level equal those of its projection
    onto level 0 (Eq.1, Eq.16: the hierarchy preserves the objective);
  * each level removes exactly its matched pairs: N_{l+1} = N_l - matched_l."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests import _pins

CASES = [
    ("C1", lambda: hgpgen.tiny(1), 16, 32),
    ("C1-w3", lambda: hgpgen.tiny(2, wmax_n=3), 16, 32),
    ("snn-small", lambda: hgpgen.snn(5, layers=4, rows=10, cols=10, fanout=15, window=5, rewire=0.1), 16, 64),
    ("vlsi-small", lambda: hgpgen.vlsi(6, 500, 500, dmax=60, in_cap=40), 16, 64),
    ("kway", lambda: hgpgen.vlsi(7, 300, 300, dmax=30, in_cap=1000), 155, ref.UNBOUNDED),
]


@pytest.mark.parametrize("name,make,omega,delta", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("cap,leftover", [(0, False), (1 << 22, False), (1 << 22, True)])
def test_hierarchy_invariants(name, make, omega, delta, cap, leftover):
    hg = make()
    g0 = ref.build_csr_hg(hg)
    r = ref.coarsen(g0, ref.params(omega, delta, 4, noise_seed=3, noise_cap=cap), leftover=leftover)
    levels, rho, gl = r["levels"], r["rho"], r["coarsest"]
    W = int(hg.node_w.astype(np.int64).sum())
    stop = 1 if omega == ref.UNBOUNDED else -(-W // omega)
    assert r["stop_nodes"] == stop
    # stop rule: the last level stops, no earlier one does
    last = levels[-1]
    # (a level that formed no pair, by a4 or by f2, has N' = N)
    assert last["Nc"] <= stop or last["Nc"] == last["N"] or len(levels) == 64
    for lv in levels[:-1]:
        assert lv["Nc"] > stop and lv["Nc"] < lv["N"]
    # N_{l+1} = N_l - pairs formed (a4 pairs, plus f2 pairs with leftover), and levels chain
    for a, b in zip(levels, levels[1:]):
        assert b["N"] == a["Nc"] and b["E"] == a["Ec"] and b["P"] == a["Pc"]
    for lv in levels:
        pairs = int(np.count_nonzero(lv["match"] != ref.NONE)) // 2
        assert lv["Nc"] == lv["N"] - pairs
        if not leftover:
            assert pairs == sum(lv["matched_per_round"])
    assert len(levels) >= 2
    # rho onto [0, N_L); sizes conserved; Omega / Delta on the original edges
    Nl = gl.N
    assert rho.shape == (g0.N,) and int(rho.max()) == Nl - 1 and len(np.unique(rho)) == Nl
    assert np.array_equal(gl.node_w.astype(np.int64), np.bincount(rho, weights=hg.node_w, minlength=Nl).astype(np.int64))
    assert int(gl.node_w.max()) <= omega
    edges0 = _pins.edges_of(g0.edge_off, g0.edge_nsrc, g0.pins)
    inb = _pins.inbound_counts(edges0, np.ones(g0.E, dtype=np.int64), rho, Nl)
    assert list(gl.in_mu) == inb
    if delta != ref.UNBOUNDED:
        assert max(inb) <= delta
    # objective preserved through the hierarchy
    edgesl = _pins.edges_of(gl.edge_off, gl.edge_nsrc, gl.pins)
    rng = np.random.default_rng(11)
    for k in (1, 2, 3, max(2, Nl // 4)):
        rc = rng.integers(0, k, size=Nl)
        assert _pins.connectivity(edgesl, gl.edge_w, rc) == _pins.connectivity(edges0, g0.edge_w, rc[rho])
        assert _pins.cut_net(edgesl, gl.edge_w, rc) == _pins.cut_net(edges0, g0.edge_w, rc[rho])
