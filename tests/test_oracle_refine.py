"""Oracle of the rows after the level pinned against brute force and SPEC examples:
f1 partition quality (Eq.1, Eq.16, constraint loads), f3 pins matrix / Eq.13 proposals / in-sequence
gains (Eqs.14-15), f4 per-move violation counts and the landing point.

Every brute force here recomputes from scratch with plain Python sets (tests/_pins.py): Eq.1 via
_pins.connectivity on the partition after the move(s), sizes and mu-weighted inbound counts via
_pins.inbound_counts — none of it shares the oracle's incremental bookkeeping."""
import json
import os
from collections import Counter

import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests import _pins

NONE = ref.NONE
HERE = os.path.dirname(__file__)


def h_ex():
    gd = json.load(open(os.path.join(HERE, "golden", "h_ex.json")))["graph"]
    return ref.build_csr(gd["num_nodes"], np.array(gd["edge_off"], dtype=np.uint64),
                         np.array(gd["edge_nsrc"], dtype=np.uint32), np.array(gd["pins"], dtype=np.uint32),
                         np.array(gd["edge_w"], dtype=np.uint32), np.array(gd["node_w"], dtype=np.uint32))


def graphs():
    yield "tiny-80", hgpgen.tiny(41, num_nodes=80, num_edges=200, size_binom=5, in_cap=12, wmax_e=5, wmax_n=3)
    yield "snn-small", hgpgen.snn(42, layers=3, rows=6, cols=6, fanout=8, window=3, rewire=0.2)
    yield "vlsi-small", hgpgen.vlsi(43, 150, 150, dmax=20, in_cap=20)


def edges_and_sizes(g):
    return _pins.edges_of(g.edge_off, g.edge_nsrc, g.pins), [int(x) for x in g.node_w]


def test_h_ex_spec_examples():
    """S: propose_moves example on H_ex, rho = {0,1}|{2,3}: node 2 -> p0 has saving 3 (e0, e1 each
    leave one pin), loss 1 (e2 absent from p0), gain 2; applying it drops Eq.1 from 3 to 1."""
    g = h_ex()
    met = json.load(open(os.path.join(HERE, "golden", "h_ex.json")))["metrics"]   # S:73-81 values
    part = met["rho"]
    q = ref.partition_metrics(g, part, 2)
    assert q["connectivity"] == met["connectivity"] == 3 and q["cut_net"] == met["cut_net"] == 3
    assert ref.partition_metrics(g, [0, 1, 2, 3], 4)["connectivity"] == met["connectivity_singletons"]
    dest, gain = ref.propose_moves(g, part, 2)
    assert dest[2] == 0 and gain[2] == 2
    assert ref.in_sequence_gains(g, part, 2, [2], dest).tolist() == [2]
    assert ref.partition_metrics(g, [0, 0, 0, 1], 2)["connectivity"] == 1
    # f4: in(2) = {e0, e1}; moving 2 to p0 makes p0 hold both inbound edges of 2 (plus e0's dst 1)
    assert ref.sequence_violations(g, part, 2, [2], dest, 3, 1).tolist() == [1]   # p0 now has 2 inbound
    assert ref.sequence_violations(g, part, 2, [2], dest, 3, 2).tolist() == [0]


def test_spec_overfill_then_vacate():
    """S: validate_sequence example: a move overfilling p_d then a second move vacating it gives
    violation counts [1, 0]; only position 2 is a legal landing point."""
    g = h_ex()
    part = [0, 0, 1, 1]                                  # sizes 2 | 2, Omega = 2
    dest = np.array([1, NONE, 0, NONE], dtype=np.uint32)
    seq = [0, 2]                                        # 0: p0 -> p1 (p1 = 3 > 2), then 2: p1 -> p0
    assert ref.sequence_violations(g, part, 2, seq, dest, 2, ref.UNBOUNDED).tolist() == [1, 0]
    gs = ref.in_sequence_gains(g, part, 2, seq, dest)
    k, best = ref.best_prefix(gs, [1, 0])
    assert (k == 2) == (gs.sum() > 0) and (k == 0 or best == gs.sum())


@pytest.mark.parametrize("name,hg", list(graphs()), ids=lambda x: x if isinstance(x, str) else "")
@pytest.mark.parametrize("nparts", [2, 5])
def test_refine_rows_against_bruteforce(name, hg, nparts):
    g = ref.build_csr_hg(hg)
    edges, sizes = edges_and_sizes(g)
    rng = np.random.default_rng(nparts + len(name))
    part = rng.integers(0, nparts, size=g.N).astype(np.uint32)
    mu = [int(x) for x in g.edge_mu]
    # ---- f1: Eq.1 / Eq.16 / loads
    q = ref.partition_metrics(g, part, nparts, omega=int(np.bincount(part, weights=sizes).max()) - 1, delta=5)
    assert q["connectivity"] == _pins.connectivity(edges, g.edge_w, part)
    assert q["cut_net"] == _pins.cut_net(edges, g.edge_w, part)
    psize = np.bincount(part, weights=sizes, minlength=nparts).astype(np.int64)
    inb = _pins.inbound_counts(edges, mu, part, nparts)
    assert q["max_size"] == psize.max() and q["max_inbound"] == max(inb)
    assert q["size_violations"] == int((psize > psize.max() - 1).sum()) and q["inbound_violations"] == sum(x > 5 for x in inb)
    # ---- f3: pins(p, e) and pins_in(p, e) (Σ_p pins = |e|, Σ_p pins_in = |dst(e)|)
    for inbound in (False, True):
        off, pp, cc = ref.pins_matrix(g, part, inbound)
        for e, (S, D) in enumerate(edges):
            want = Counter(int(part[x]) for x in (D if inbound else S | D))
            got = dict(zip(pp[off[e]:off[e + 1]].tolist(), cc[off[e]:off[e + 1]].tolist()))
            assert got == dict(want) and list(got) == sorted(got)
    # ---- f3: Eq.13 gain(n, p) = Eq.1 before - Eq.1 after moving n alone to p; best = max (gain, p)
    base = _pins.connectivity(edges, g.edge_w, part)
    for enforce in (False, True):
        omega = int(psize.max()) + 1
        dest, gain = ref.propose_moves(g, part, nparts, omega=omega, enforce_size=enforce)
        for n in range(g.N):
            inc = [e for e, (S, D) in enumerate(edges) if n in S or n in D]
            cands = {int(part[x]) for e in inc for x in edges[e][0] | edges[e][1]} - {int(part[n])}
            if enforce:
                cands = {p for p in cands if sizes[n] + psize[p] <= omega}
            best = None
            for p in sorted(cands):
                moved = part.copy()
                moved[n] = p
                gp = base - _pins.connectivity(edges, g.edge_w, moved)
                if best is None or (gp, p) > best:
                    best = (gp, p)
            assert (int(dest[n]), int(gain[n])) == ((NONE, 0) if best is None else (best[1], best[0])), n
    # ---- f3 in-sequence gains and f4 violations on a sequence of the proposals (gain order)
    dest, gain = ref.propose_moves(g, part, nparts)
    movers = [n for n in range(g.N) if dest[n] != NONE]
    seq = sorted(movers, key=lambda n: (-int(gain[n]), n))
    gs = ref.in_sequence_gains(g, part, nparts, seq, dest)
    omega, delta = int(psize.max()), max(inb)
    vio = ref.sequence_violations(g, part, nparts, seq, dest, omega, delta)
    cur = part.copy()
    conn = base
    for i, n in enumerate(seq):
        cur[n] = dest[n]
        c2 = _pins.connectivity(edges, g.edge_w, cur)
        assert gs[i] == conn - c2, i                      # Σ prefix gains = Eq.1 change
        conn = c2
        sz = np.bincount(cur, weights=sizes, minlength=nparts)
        ib = _pins.inbound_counts(edges, mu, cur, nparts)
        assert vio[i] == sum(1 for p in range(nparts) if sz[p] > omega or ib[p] > delta), i
    # in-sequence = in-isolation for the first move (S: "sequence of 1 move")
    if seq:
        assert gs[0] == gain[seq[0]]
    # landing point by enumeration (ties -> shortest; nothing unless > 0)
    k, best = ref.best_prefix(gs, vio)
    cands = [(int(gs[:j + 1].sum()), -(j + 1)) for j in range(len(seq)) if vio[j] == 0]
    top = max(cands, default=(0, 0))
    assert (k, best) == ((-top[1], top[0]) if top[0] > 0 else (0, 0))


def test_in_sequence_swap_and_shared_departure():
    """S: in_sequence_gains examples: a swap of the two pins of an edge; two pins of one 2-pin edge
    leaving their shared partition to different partitions, where the later move's gain differs
    from its in-isolation gain. Checked against Eq.1 recomputation and values derived by hand."""
    # nodes 0,1 in p0, node 2 in p1, node 3 in p2; edge e0 = {0 -> 1}, e1 = {0 -> 2}, e2 = {1 -> 3}
    g = ref.build_csr(4, np.array([0, 2, 4, 6], dtype=np.uint64), np.array([1, 1, 1], dtype=np.uint32),
                      np.array([0, 1, 0, 2, 1, 3], dtype=np.uint32), np.array([1, 1, 1], dtype=np.uint32),
                      np.ones(4, dtype=np.uint32))
    edges = _pins.edges_of(g.edge_off, g.edge_nsrc, g.pins)
    part = np.array([0, 0, 1, 2], dtype=np.uint32)
    dest = np.array([1, 2, NONE, NONE], dtype=np.uint32)
    gs = ref.in_sequence_gains(g, part, 3, [0, 1], dest)
    iso = []
    for n in (0, 1):
        m = part.copy()
        m[n] = dest[n]
        iso.append(_pins.connectivity(edges, g.edge_w, part) - _pins.connectivity(edges, g.edge_w, m))
    after = part.copy()
    after[0], after[1] = 1, 2
    assert gs.sum() == _pins.connectivity(edges, g.edge_w, part) - _pins.connectivity(edges, g.edge_w, after)
    # by hand: conn 2 -> 2 (0 leaves e1's p0 side, opens e0) -> 1 (1 joins 3 in p2 and is e0's last
    # pin in its old part): in-sequence [0, 1] although node 1 gains 0 in isolation
    assert gs.tolist() == [0, 1] and iso == [0, 0]
    swap = np.array([1, 0, NONE, NONE], dtype=np.uint32)
    part2 = np.array([0, 1, 1, 2], dtype=np.uint32)
    gs2 = ref.in_sequence_gains(g, part2, 3, [0, 1], swap)
    fin = part2.copy()
    fin[0], fin[1] = 1, 0
    assert gs2.sum() == _pins.connectivity(edges, g.edge_w, part2) - _pins.connectivity(edges, g.edge_w, fin)
