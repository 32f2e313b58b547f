"""GPU (libhgp.so through the C-ABI) vs the CPU oracle, step by step and over several levels."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import assert_cand_equal, assert_csr_equal, assert_nbrs_equal, dev, gpu_build

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


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


def _cases():
    return [
        ("C1-s1", lambda: hgpgen.tiny(1), 16, 32, dict(noise=True)),
        ("C1-s2-w3", lambda: hgpgen.tiny(2, wmax_n=3), 16, 32, dict(noise=False)),
        ("C1-s3-norm1", lambda: hgpgen.tiny(3), 16, 32, dict(norm=1)),
        ("dense", lambda: hgpgen.tiny(4, num_nodes=300, num_edges=3000, size_binom=8, in_cap=200), 8, 200, dict()),
        ("snn-small", lambda: hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30, window=9, rewire=0.1), 16, 256,
         dict()),
        ("vlsi-small", lambda: hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600), 64, 600, dict()),
        ("kway", lambda: hgpgen.vlsi(7, 5000, 5000, dmax=200, in_cap=10 ** 6), 2575, hgpgen.UNBOUNDED, dict(pi=2)),
        ("pi16", lambda: hgpgen.tiny(8, num_nodes=400, num_edges=2000), 16, 40, dict(pi=16)),
        ("pi1", lambda: hgpgen.tiny(9), 16, 32, dict(pi=1)),
    ]


@pytest.mark.parametrize("name,make,omega,delta,kw", _cases(), ids=[c[0] for c in _cases()])
def test_level_steps_match_oracle(hgp, ctx, name, make, omega, delta, kw):
    hg = make()
    pi = kw.get("pi", 4)
    norm = kw.get("norm", 0)
    cap = hgpgen.default_noise_cap(hg) if kw.get("noise", True) else 0
    # a1
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    assert_csr_equal(g.to_host(), rg, "a1")
    # a2
    nb = hgp.unique_neighbors(ctx, g)
    rnb = ref.unique_neighbors(rg)
    assert_nbrs_equal(nb.to_host(), rnb, "a2")
    for level in range(3):
        p = hgp.params(omega, delta, pi, norm=norm, noise_seed=level + 11, noise_cap=cap)
        rp = ref.params(omega, delta, pi, norm=norm, noise_seed=level + 11, noise_cap=cap)
        # a3
        cand = hgp.empty_cand(g.N, pi)
        hgp.score_pairs(ctx, g, nb, p, cand)
        rcand = ref.score_pairs(rg, rnb, rp)
        assert_cand_equal(hgp.cand_to_numpy(cand), rcand)
        assert_nbrs_equal(nb.to_host(), rnb, f"a3 flags level {level}")
        # a4 (same candidates on both sides)
        m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
        per = torch.zeros(pi, dtype=torch.uint32, device="cuda")
        hgp.match(ctx, cand, g.N, pi, m, per)
        rm, rper, _ = ref.match(rcand, pi)
        assert np.array_equal(m.cpu().numpy(), rm), f"a4 match differs at level {level}"
        assert np.array_equal(per.cpu().numpy(), rper)
        # a5
        gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
        cg, cnb = hgp.contract(ctx, g, nb, m, gam)
        rgam, rcg, rcnb = ref.contract(rg, rnb, rm)
        assert np.array_equal(gam.cpu().numpy(), rgam)
        assert_csr_equal(cg.to_host(), rcg, f"a5 level {level}")
        assert_nbrs_equal(cnb.to_host(), rcnb, f"a5 nbrs level {level}")
        g, nb, rg, rnb = cg, cnb, rcg, rcnb
        if g.N < 2:
            break


def test_coarsen_level_composition(hgp, ctx):
    hg = hgpgen.tiny(12)
    g = gpu_build(hgp, ctx, hg)
    nb = hgp.unique_neighbors(ctx, g)
    p = hgp.params(16, 32, 4, noise_seed=1, noise_cap=1 << 22)
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cand = hgp.empty_cand(g.N, 4)
    cg, cnb, st = hgp.coarsen_level(ctx, g, nb, p, cand, m, gam)
    rg = ref.build_csr_hg(hg)
    rnb = ref.unique_neighbors(rg)
    rr = ref.coarsen_level(rg, rnb, ref.params(16, 32, 4, noise_seed=1, noise_cap=1 << 22))
    assert_cand_equal(hgp.cand_to_numpy(cand), rr["cand"])
    assert np.array_equal(m.cpu().numpy(), rr["match"])
    assert np.array_equal(gam.cpu().numpy(), rr["gamma"])
    assert_csr_equal(cg.to_host(), rr["coarse"])
    assert_nbrs_equal(cnb.to_host(), rr["coarse_nb"])
    assert st["Nc"] == rr["coarse"].N and st["Ec"] == rr["coarse"].E
    assert st["matched_per_round"] == list(rr["matched_per_round"])
    assert st["ms"]["total"] > 0


def test_deterministic_reruns(hgp, ctx):
    """Two runs on the same input give identical bytes (sets compared sorted)."""
    hg = hgpgen.vlsi(3, 30000, 30000, dmax=512, in_cap=800)
    outs = []
    for _ in range(2):
        g = gpu_build(hgp, ctx, hg)
        nb = hgp.unique_neighbors(ctx, g)
        p = hgp.params(64, 800, 4, noise_seed=5, noise_cap=1 << 22)
        m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
        gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
        cand = hgp.empty_cand(g.N, 4)
        cg, cnb, _ = hgp.coarsen_level(ctx, g, nb, p, cand, m, gam)
        h = cg.to_host()
        nbh = cnb.to_host()
        order = np.lexsort((nbh["nbr"], np.repeat(np.arange(len(nbh["off"]) - 1), np.diff(nbh["off"].astype(np.int64)))))
        outs.append((cand.cpu().numpy(), m.cpu().numpy(), gam.cpu().numpy(), h, nbh["off"], nbh["nbr"][order]))
    a, b = outs
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    for k in a[3]:
        assert np.array_equal(a[3][k], b[3][k]), k
    assert np.array_equal(a[4], b[4]) and np.array_equal(a[5], b[5])


@pytest.mark.parametrize("bad,code,idx", [
    (dict(edge_off=[0, 2, 2], edge_nsrc=[1, 0], pins=[0, 1]), -2, "edge 1"),
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 1], pins=[0, 1, 2, 2]), -2, "edge 1"),
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 1], pins=[0, 1, 1, 1]), -2, "edge 1"),
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 3], pins=[0, 1, 1, 2]), -2, "edge 1"),
    (dict(edge_off=[0, 2, 4], edge_nsrc=[1, 1], pins=[0, 1, 1, 9]), -2, "edge 1"),
    (dict(edge_off=[0, 3, 1], edge_nsrc=[1, 0], pins=[0, 1, 2]), -2, "edge 1"),
])
def test_malformed_inputs_match_oracle(hgp, ctx, bad, code, idx):
    E = len(bad["edge_nsrc"])
    args = (np.array(bad["edge_off"], dtype=np.uint64), np.array(bad["edge_nsrc"], dtype=np.uint32),
            np.array(bad["pins"], dtype=np.uint32), np.ones(E, dtype=np.uint32), np.ones(4, dtype=np.uint32))
    with pytest.raises(hgp.HgpError) as eg:
        hgp.build_csr(ctx, 4, *[dev(a) for a in args])
    with pytest.raises(ref.OracleError) as eo:
        ref.build_csr(4, *args)
    assert eg.value.code == eo.value.code == code
    assert idx in eg.value.msg and idx in eo.value.msg


def test_infeasible_and_weights(hgp, ctx):
    hg = hgpgen.tiny(1)
    g = gpu_build(hgp, ctx, hg)
    nb = hgp.unique_neighbors(ctx, g)
    cand = hgp.empty_cand(g.N, 4)
    with pytest.raises(hgp.HgpError) as e:
        hgp.score_pairs(ctx, g, nb, hgp.params(16, 3, 4), cand)
    rg = ref.build_csr_hg(hg)
    rnb = ref.unique_neighbors(rg)
    with pytest.raises(ref.OracleError) as eo:
        ref.score_pairs(rg, rnb, ref.params(16, 3, 4))
    assert e.value.code == eo.value.code == -3
    assert e.value.msg.split(":")[0] == eo.value.msg.split(":")[0]


def test_empty_and_isolated(hgp, ctx):
    # no edges at all; isolated nodes contract to themselves
    z64, z32 = np.zeros(1, dtype=np.uint64), np.zeros(0, dtype=np.uint32)
    g = hgp.build_csr(ctx, 5, dev(z64), dev(z32), dev(z32), dev(z32), dev(np.ones(5, dtype=np.uint32)))
    nb = hgp.unique_neighbors(ctx, g)
    assert nb.V == 0
    m = torch.empty(5, dtype=torch.uint32, device="cuda")
    gam = torch.empty(5, dtype=torch.uint32, device="cuda")
    cg, cnb, st = hgp.coarsen_level(ctx, g, nb, hgp.params(4, 4, 4), None, m, gam)
    assert st["Nc"] == 5 and st["Ec"] == 0
    assert list(gam.cpu().numpy()) == [0, 1, 2, 3, 4]


def test_giant_edges_and_hubs(hgp, ctx):
    """Edges above the warp (1024) and CTA (16384) sort tiers, neighbourhoods above every
    shared-memory tier of a2/a3/a5."""
    rng = np.random.default_rng(0)
    N = 40000
    sizes = [20000, 3000, 1500, 40, 2] + [int(x) for x in rng.integers(2, 30, size=3000)]
    pins, nsrc, off = [], [], [0]
    for s in sizes:
        p = rng.choice(N, size=s, replace=False)
        pins.extend(p.tolist())
        nsrc.append(int(rng.integers(0, 3)) if s > 2 else 1)
        off.append(len(pins))
    hg = hgpgen.Hypergraph(N, np.array(off, dtype=np.uint64), np.array(nsrc, dtype=np.uint32),
                           np.array(pins, dtype=np.uint32), np.ones(len(sizes), dtype=np.uint32),
                           np.ones(N, dtype=np.uint32))
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    assert_csr_equal(g.to_host(), rg, "a1 giant")
    nb = hgp.unique_neighbors(ctx, g)
    rnb = ref.unique_neighbors(rg)
    assert_nbrs_equal(nb.to_host(), rnb, "a2 giant")
    p = hgp.params(8, 10 ** 6, 4, noise_seed=3, noise_cap=1 << 20)
    cand = hgp.empty_cand(g.N, 4)
    hgp.score_pairs(ctx, g, nb, p, cand)
    rcand = ref.score_pairs(rg, rnb, ref.params(8, 10 ** 6, 4, noise_seed=3, noise_cap=1 << 20))
    assert_cand_equal(hgp.cand_to_numpy(cand), rcand)
    assert_nbrs_equal(nb.to_host(), rnb, "a3 giant flags")
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    hgp.match(ctx, cand, g.N, 4, m, None)
    rm, _, _ = ref.match(rcand, 4)
    assert np.array_equal(m.cpu().numpy(), rm)
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cg, cnb = hgp.contract(ctx, g, nb, m, gam)
    rgam, rcg, rcnb = ref.contract(rg, rnb, rm)
    assert_csr_equal(cg.to_host(), rcg, "a5 giant")
    assert_nbrs_equal(cnb.to_host(), rcnb, "a5 giant nbrs")


def test_long_chain_pointer_jumping(hgp, ctx):
    """A path 0-1-...-n with equal weights and no noise: every node targets its higher
    neighbour, giving one chain of length ~n (beyond the walk cap) — a4 must still equal the DP."""
    n = 3000
    off = np.arange(0, 2 * n + 1, 2, dtype=np.uint64)
    pins = np.stack([np.arange(n), np.arange(1, n + 1)], axis=1).reshape(-1).astype(np.uint32)
    # weights increasing along the path keep every child's gain > 0 (Eqs.9-10), so the best-child
    # chain is the whole path (with equal weights the gains alternate to 0 and chains stay short)
    hg = hgpgen.Hypergraph(n + 1, off, np.zeros(n, dtype=np.uint32), pins, np.arange(1, n + 1, dtype=np.uint32),
                           np.ones(n + 1, dtype=np.uint32))
    g = gpu_build(hgp, ctx, hg)
    nb = hgp.unique_neighbors(ctx, g)
    cand = hgp.empty_cand(g.N, 4)
    hgp.score_pairs(ctx, g, nb, hgp.params(2, 10, 4), cand)
    rg = ref.build_csr_hg(hg)
    rnb = ref.unique_neighbors(rg)
    rcand = ref.score_pairs(rg, rnb, ref.params(2, 10, 4))
    assert_cand_equal(hgp.cand_to_numpy(cand), rcand)
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    hgp.match(ctx, cand, g.N, 4, m, None)
    rm, _, _ = ref.match(rcand, 4)
    assert np.array_equal(m.cpu().numpy(), rm)
    assert ctx.tier_counts()["jump"] > 0, "the chain must reach a4's pointer-jumping fallback"


FUSED_CASES = [
    ("snn-small", lambda: hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30, window=9, rewire=0.1), 16, 256),
    ("snn-model", lambda: hgpgen.snn(6, layers=3, rows=30, cols=30, fanout=60, window=11), 64, 4096),
    ("C1", lambda: hgpgen.tiny(1), 16, 32),
    ("vlsi-small", lambda: hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600), 64, 600),
    ("kway", lambda: hgpgen.vlsi(7, 5000, 5000, dmax=200, in_cap=10 ** 6), 2575, hgpgen.UNBOUNDED),
]


@pytest.mark.parametrize("name,make,omega,delta", FUSED_CASES, ids=[c[0] for c in FUSED_CASES])
def test_fused_level0_matches_oracle(hgp, ctx, name, make, omega, delta):
    """hgp_coarsen_level0 (fused a2+a3 when representable) == oracle a2, a3, a4, a5."""
    hg = make()
    cap = hgpgen.default_noise_cap(hg)
    g = gpu_build(hgp, ctx, hg)
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cand = hgp.empty_cand(g.N, 4)
    ctx.profile_begin("nbr")
    nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap), cand, m, gam)
    ctx.profile_end()
    used = ctx.profile_report()
    rg = ref.build_csr_hg(hg)
    rnb = ref.unique_neighbors(rg)
    rr = ref.coarsen_level(rg, rnb, ref.params(omega, delta, 4, noise_seed=2, noise_cap=cap))
    assert_nbrs_equal(nb.to_host(), rnb, "fused nbrs+flags")
    assert_cand_equal(hgp.cand_to_numpy(cand), rr["cand"])
    assert np.array_equal(m.cpu().numpy(), rr["match"])
    assert np.array_equal(gam.cpu().numpy(), rr["gamma"])
    assert_csr_equal(cg.to_host(), rr["coarse"], "fused coarse")
    assert_nbrs_equal(cnb.to_host(), rr["coarse_nb"], "fused coarse nbrs")
    if name.startswith("snn"):   # uniform edge weights: the fused kernel handles every node
        assert "nbrscore_A" in used and "nbrs_t1" not in used, used
    # without returning N(n) (a5 reads it from the fused kernel's pool): same level
    m2 = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    gam2 = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cand2 = hgp.empty_cand(g.N, 4)
    nb2, cg2, cnb2, st2 = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap), cand2,
                                             m2, gam2, want_nbrs=False)
    assert nb2 is None and st2["V"] == rnb.nbr.shape[0]
    assert np.array_equal(m2.cpu().numpy(), rr["match"]) and np.array_equal(gam2.cpu().numpy(), rr["gamma"])
    assert_csr_equal(cg2.to_host(), rr["coarse"], "fused coarse (pool view)")
    assert_nbrs_equal(cnb2.to_host(), rr["coarse_nb"], "fused coarse nbrs (pool view)")


@pytest.mark.parametrize("mode", ["pool64", "pool1", "unfused"])
@pytest.mark.parametrize("name,make,omega,delta", FUSED_CASES[1:], ids=[c[0] for c in FUSED_CASES[1:]])
def test_fused_level0_partial_paths(hgp, ctx, monkeypatch, mode, name, make, omega, delta):
    """The fused call's secondary paths give the same level: a first pool too small for most nodes
    (second, exact pool), and every node on the unfused list path (k_nbrs + k_score over the
    segment view) — both with and without returning N(n)."""
    opts = {"fused_pool_cap": int(mode[4:])} if mode.startswith("pool") else {"unfused": 1}
    with ctx.options(**opts):
        _partial_paths(hgp, ctx, mode, make, omega, delta)


def _partial_paths(hgp, ctx, mode, make, omega, delta):
    hg = make()
    cap = hgpgen.default_noise_cap(hg)
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    rnb = ref.unique_neighbors(rg)
    rr = ref.coarsen_level(rg, rnb, ref.params(omega, delta, 4, noise_seed=2, noise_cap=cap))
    for want in (True, False):
        m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
        gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
        cand = hgp.empty_cand(g.N, 4)
        ctx.profile_begin("nbr")
        nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap), cand,
                                             m, gam, want_nbrs=want)
        ctx.profile_end()
        used = ctx.profile_report()
        if mode == "unfused":
            assert "nbrscore_A" not in used and "nbrs_list_t1" in used, used
        if want:
            assert_nbrs_equal(nb.to_host(), rnb, f"{mode} nbrs+flags")
        assert st["V"] == rnb.nbr.shape[0]
        assert_cand_equal(hgp.cand_to_numpy(cand), rr["cand"])
        assert np.array_equal(m.cpu().numpy(), rr["match"])
        assert np.array_equal(gam.cpu().numpy(), rr["gamma"])
        assert_csr_equal(cg.to_host(), rr["coarse"], f"{mode} coarse")
        assert_nbrs_equal(cnb.to_host(), rr["coarse_nb"], f"{mode} coarse nbrs")


@pytest.mark.parametrize("name,make", [("C1", lambda: hgpgen.tiny(1)), ("tiny-N", lambda: hgpgen.tiny(3, num_nodes=100, num_edges=200)),
                                       ("vlsi-small", lambda: hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600)),
                                       ("snn-small", lambda: hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30,
                                                                         window=9, rewire=0.1))])
def test_radix_incidence_matches_oracle(hgp, ctx, monkeypatch, name, make):
    """a1 with the radix-sort transpose (option inc_radix; 1, 2 or 3 passes by node count) builds the
    same canonical incidence as the oracle, and so does a5's coarse incidence."""
    with ctx.options(inc_radix=1):
        _radix(hgp, ctx, make)


def _radix(hgp, ctx, make):
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    assert_csr_equal(g.to_host(), rg, "a1 (radix)")
    nb = hgp.unique_neighbors(ctx, g)
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cg, cnb, _ = hgp.coarsen_level(ctx, g, nb, hgp.params(64, 600, 4), None, m, gam)
    rr = ref.coarsen_level(rg, ref.unique_neighbors(rg), ref.params(64, 600, 4))
    assert_csr_equal(cg.to_host(), rr["coarse"], "a5 (radix)")


@pytest.mark.parametrize("name,make,frac", [
    ("snn-rand-big-nbhd", lambda: hgpgen.snn(8, layers=4, rows=40, cols=60, fanout=99, window=15, rewire=1.0), True),
    ("vlsi-small", lambda: hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600), False),
])
def test_fused_level0_sampled_first_tier(hgp, ctx, monkeypatch, name, make, frac):
    """The fused call samples every 64th node in tier A first and starts the rest in tier M when
    most samples overflow A's table (option fused_sample_min lowers the size at which it samples):
    the level is the same either way."""
    with ctx.options(fused_sample_min=128):
        _sampled(hgp, ctx, name, make, frac)


def _sampled(hgp, ctx, name, make, frac):
    hg = make()
    cap = hgpgen.default_noise_cap(hg)
    omega, delta = (256, 4096) if name.startswith("snn") else (64, 600)
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    rnb = ref.unique_neighbors(rg)
    rr = ref.coarsen_level(rg, rnb, ref.params(omega, delta, 4, noise_seed=2, noise_cap=cap))
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cand = hgp.empty_cand(g.N, 4)
    ctx.profile_begin("nbr")
    nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap), cand, m, gam)
    ctx.profile_end()
    used = ctx.profile_report()
    assert ("nbrscore_M" in used) == frac or not frac, used
    assert_nbrs_equal(nb.to_host(), rnb, "sampled nbrs+flags")
    assert_cand_equal(hgp.cand_to_numpy(cand), rr["cand"])
    assert np.array_equal(gam.cpu().numpy(), rr["gamma"])
    assert_csr_equal(cg.to_host(), rr["coarse"], "sampled coarse")
    assert_nbrs_equal(cnb.to_host(), rr["coarse_nb"], "sampled coarse nbrs")
