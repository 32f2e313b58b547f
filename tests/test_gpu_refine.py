"""GPU rows after the level vs the oracle (oracle/hgp_ref_refine.cpp), bit for bit:
f1 partition quality (Eq.1, Eq.16, loads and violation counts), f3 the
pins(p, e) / pins_in(p, e) matrices, Eq.13 proposals
and in-sequence gains (Eqs.14-15), f4 per-move violation counts of the event-based
checks and the landing point. Partitions are random (few and many parts) and the
initial partition rho of the multi-level driver; sequences are the proposals in
gain order (the chained order of P:944-960 is not part of these rows)."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import dev, gpu_build

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
NONE = ref.NONE


@pytest.fixture(scope="module")
def hgp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_20497_b200 import hgp as h
    h.lib()
    return h


@pytest.fixture(scope="module")
def ctx(hgp):
    return hgp.Ctx(0)


GRAPHS = [
    ("tiny-80", lambda: hgpgen.tiny(41, num_nodes=80, num_edges=200, size_binom=5, in_cap=12, wmax_e=5, wmax_n=3)),
    ("C1", lambda: hgpgen.tiny(1)),
    ("snn-small", lambda: hgpgen.snn(42, layers=3, rows=6, cols=6, fanout=8, window=3, rewire=0.2)),
    ("snn-mid", lambda: hgpgen.snn(7, layers=4, rows=20, cols=25, fanout=40, window=9, rewire=0.1)),
    # hub nodes: sum over I(n) of |row(e)| > 512 with many parts (the CTA tier of the proposals)
    ("vlsi-hubs", lambda: hgpgen.vlsi(43, 3000, 3000, dmax=300, in_cap=200)),
]


def _sequence(dest, gain):
    movers = np.nonzero(dest != NONE)[0]
    order = np.lexsort((movers, -gain[movers].astype(np.int64)))
    return movers[order].astype(np.uint32)


@pytest.mark.parametrize("nparts_rule", ["2", "7", "N/3"])
@pytest.mark.parametrize("name,make", GRAPHS, ids=[g[0] for g in GRAPHS])
def test_refine_rows_match_oracle(hgp, ctx, name, make, nparts_rule):
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    N = rg.N
    nparts = {"2": 2, "7": 7, "N/3": max(2, N // 3)}[nparts_rule]
    rng = np.random.default_rng(len(name) * 31 + nparts)
    part = rng.integers(0, nparts, size=N).astype(np.uint32)
    pt = dev(part)
    sizes = np.bincount(part, weights=rg.node_w, minlength=nparts).astype(np.int64)
    omega = int(sizes.max())
    # ---- pins / pins_in
    for inbound in (False, True):
        pm = hgp.pins_matrix(ctx, g, pt, nparts, inbound).to_host()
        off, pp, cc = ref.pins_matrix(rg, part, inbound)
        assert np.array_equal(pm["off"], off) and np.array_equal(pm["part"], pp) and np.array_equal(pm["count"], cc)
    # ---- f1 quality, with limits that make some partitions violate
    q_ref = ref.partition_metrics(rg, part, nparts, omega - 1, 3)
    q, size, inb = hgp.partition_metrics(ctx, g, pt, nparts, omega - 1, 3, loads=True)
    assert q == q_ref
    assert int(size.cpu().numpy().max()) == q_ref["max_size"]
    # ---- f3 Eq.13 proposals, with and without the size filter
    pins = hgp.pins_matrix(ctx, g, pt, nparts)
    for enforce, om in ((False, ref.UNBOUNDED), (True, omega + 1)):
        d_ref, g_ref = ref.propose_moves(rg, part, nparts, omega=om, enforce_size=enforce)
        d, gn = hgp.propose_moves(ctx, g, pt, nparts, om, enforce, pins=pins if enforce else None)
        assert np.array_equal(d.cpu().numpy(), d_ref), f"dest differs at {np.nonzero(d.cpu().numpy() != d_ref)[0][:5]}"
        assert np.array_equal(gn.cpu().numpy(), g_ref)
    # ---- f3 in-sequence gains and f4 violations on the proposals in gain order
    d_ref, g_ref = ref.propose_moves(rg, part, nparts)
    seq = _sequence(d_ref, g_ref)
    st, dt = dev(seq), dev(d_ref)
    gs_ref = ref.in_sequence_gains(rg, part, nparts, seq, d_ref)
    gs = hgp.in_sequence_gains(ctx, g, pt, nparts, st, dt, pins=pins)
    assert np.array_equal(gs.cpu().numpy(), gs_ref), f"first bad {np.nonzero(gs.cpu().numpy() != gs_ref)[0][:5]}"
    inb_max = q_ref["max_inbound"]
    for om, de in ((omega, inb_max), (omega - 1, max(inb_max - 2, 0)), (ref.UNBOUNDED, ref.UNBOUNDED)):
        v_ref = ref.sequence_violations(rg, part, nparts, seq, d_ref, om, de)
        v = hgp.sequence_violations(ctx, g, pt, nparts, st, dt, om, de)
        assert np.array_equal(v.cpu().numpy(), v_ref), f"violations differ at {np.nonzero(v.cpu().numpy() != v_ref)[0][:5]}"
        assert hgp.best_prefix(ctx, gs, v) == ref.best_prefix(gs_ref, v_ref)


@pytest.mark.parametrize("name,make,omega,delta", [
    ("C1", lambda: hgpgen.tiny(3), 16, 32),
    ("snn-mid", lambda: hgpgen.snn(8, layers=4, rows=20, cols=25, fanout=40, window=9), 64, 400),
])
def test_refine_on_the_initial_partition(hgp, ctx, name, make, omega, delta):
    """f1 on rho = gamma^L o ... o gamma^1 of the multi-level driver: quality of the
    initial partition and one refinement step (proposals -> in-sequence gains -> violations ->
    landing point), GPU vs oracle."""
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    p = hgp.params(omega, delta, 4)
    rho, coarsest, _, _ = hgp.coarsen(ctx, g, p)
    r = ref.coarsen(rg, ref.params(omega, delta, 4))
    rho_h = rho.cpu().numpy()
    assert np.array_equal(rho_h, r["rho"])
    nparts = coarsest.N
    q = hgp.partition_metrics(ctx, g, rho, nparts, omega, delta)
    assert q == ref.partition_metrics(rg, rho_h, nparts, omega, delta)
    assert q["size_violations"] == 0 and q["inbound_violations"] == 0   # coarsening keeps both limits
    d_ref, g_ref = ref.propose_moves(rg, rho_h, nparts, omega, True)
    d, gn = hgp.propose_moves(ctx, g, rho, nparts, omega, True)
    assert np.array_equal(d.cpu().numpy(), d_ref) and np.array_equal(gn.cpu().numpy(), g_ref)
    seq = _sequence(d_ref, g_ref)
    gs_ref = ref.in_sequence_gains(rg, rho_h, nparts, seq, d_ref)
    v_ref = ref.sequence_violations(rg, rho_h, nparts, seq, d_ref, omega, delta)
    gs = hgp.in_sequence_gains(ctx, g, rho, nparts, dev(seq), dev(d_ref))
    v = hgp.sequence_violations(ctx, g, rho, nparts, dev(seq), dev(d_ref), omega, delta)
    assert np.array_equal(gs.cpu().numpy(), gs_ref) and np.array_equal(v.cpu().numpy(), v_ref)
    assert hgp.best_prefix(ctx, gs, v) == ref.best_prefix(gs_ref, v_ref)


def test_refine_edge_cases(hgp, ctx):
    hg = hgpgen.tiny(2, num_nodes=50, num_edges=60)
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    part = np.zeros(rg.N, dtype=np.uint32)
    # one partition: nothing is cut, nobody can move
    q = hgp.partition_metrics(ctx, g, dev(part), 1)
    assert q["connectivity"] == 0 and q["cut_net"] == 0
    d, gn = hgp.propose_moves(ctx, g, dev(part), 1)
    assert (d.cpu().numpy() == NONE).all() and (gn.cpu().numpy() == 0).all()
    # empty sequence
    e = torch.empty(0, dtype=torch.uint32, device="cuda")
    assert hgp.in_sequence_gains(ctx, g, dev(part), 1, e, dev(part)).numel() == 0
    assert hgp.best_prefix(ctx, torch.empty(0, dtype=torch.int64, device="cuda"), e) == (0, 0)
    # a partition id out of range names the lowest such node
    bad = part.copy()
    bad[7] = 5
    bad[9] = 9
    with pytest.raises(hgp.HgpError) as ei:
        hgp.partition_metrics(ctx, g, dev(bad), 2)
    assert ei.value.code == -1 and "node 7" in ei.value.msg
    # a sequence with a duplicate node / a non-move is rejected, naming the lowest bad position
    part2 = (np.arange(rg.N) % 2).astype(np.uint32)
    dest = (1 - part2).astype(np.uint32)
    seq = np.array([3, 4, 3, 5], dtype=np.uint32)
    with pytest.raises(hgp.HgpError) as ei:
        hgp.in_sequence_gains(ctx, g, dev(part2), 2, dev(seq), dev(dest))
    assert "position 2" in ei.value.msg
    dest2 = dest.copy()
    dest2[4] = part2[4]
    with pytest.raises(hgp.HgpError) as ei:
        hgp.sequence_violations(ctx, g, dev(part2), 2, dev(np.array([3, 4], dtype=np.uint32)), dev(dest2), 10, 10)
    assert "position 1" in ei.value.msg
