"""Every kernel tier of the level is exercised by an input built for it, and on that input the
GPU equals the oracle. Tiers are read from the library's work counters (hgp_tier_counts: nodes
each tier processed), not from launch names — a launch over an empty device list counts nothing.

The last test asserts that the union over this module covers every tier of include/hgp.h."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import assert_cand_equal, assert_csr_equal, assert_nbrs_equal, gpu_build

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SEEN: dict[str, int] = {}


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


def _record(ctx):
    for k, v in ctx.tier_counts(reset=True).items():
        SEEN[k] = SEEN.get(k, 0) + v


def _hubs(seed, N, big, small=3000, smax=30, wmax=400):
    """Edges of the given (large) sizes plus many small ones: neighbourhoods above every tier."""
    rng = np.random.default_rng(seed)
    sizes = list(big) + [int(x) for x in rng.integers(2, smax, size=small)]
    pins, nsrc, off = [], [], [0]
    for s in sizes:
        pins.extend(rng.choice(N, size=s, replace=False).tolist())
        nsrc.append(int(rng.integers(0, 3)) if s > 2 else 1)
        off.append(len(pins))
    w = rng.integers(1, wmax + 1, size=len(sizes)).astype(np.uint32)
    return hgpgen.Hypergraph(N, np.array(off, dtype=np.uint64), np.array(nsrc, dtype=np.uint32),
                             np.array(pins, dtype=np.uint32), w, np.ones(N, dtype=np.uint32))


def _unfused_level(hgp, ctx, hg, omega, delta, norm=0, cap=1 << 20):
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    nb = hgp.unique_neighbors(ctx, g)
    rnb = ref.unique_neighbors(rg)
    assert_nbrs_equal(nb.to_host(), rnb, "a2")
    cand = hgp.empty_cand(g.N, 4)
    hgp.score_pairs(ctx, g, nb, hgp.params(omega, delta, 4, norm=norm, noise_seed=3, noise_cap=cap), cand)
    rcand = ref.score_pairs(rg, rnb, ref.params(omega, delta, 4, norm=norm, noise_seed=3, noise_cap=cap))
    assert_cand_equal(hgp.cand_to_numpy(cand), rcand)
    assert_nbrs_equal(nb.to_host(), rnb, "a3 flags")
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    hgp.match(ctx, cand, g.N, 4, m, None)
    rm, _, _ = ref.match(rcand, 4)
    assert np.array_equal(m.cpu().numpy(), rm)
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cg, cnb = hgp.contract(ctx, g, nb, m, gam)
    _, rcg, rcnb = ref.contract(rg, rnb, rm)
    assert_csr_equal(cg.to_host(), rcg, "a5")
    assert_nbrs_equal(cnb.to_host(), rcnb, "a5 nbrs")
    return cg, cnb, rcg, rcnb


def test_unfused_hub_tiers(hgp, ctx):
    """a2 tiers 1-3, a3 first tier and B, a5 coarse neighbour tiers A-C: edges of 20000, 7000, 3000
    and 1500 pins among many small ones."""
    ctx.tier_counts(reset=True)
    _unfused_level(hgp, ctx, _hubs(0, 30000, [17500, 7000, 3000, 1500, 40, 2]), 8, 10 ** 6)   # a5 hubs: tier H
    with ctx.options(no_hub=1):   # a3 B and H, a5 C (bounds ~18000): the tiers the hub tiers replace
        _unfused_level(hgp, ctx, _hubs(7, 12000, [9000, 3000, 40, 2], small=1000), 8, 10 ** 6)
    _record(ctx)


def test_wide_tiers(hgp, ctx):
    """norm = 1 with weights up to 400: sum c(e) over I(n) >= 2^32 -> 64-bit eta in shared memory
    (W) and, for the hub neighbourhoods, in global memory (H)."""
    ctx.tier_counts(reset=True)
    _unfused_level(hgp, ctx, _hubs(1, 20000, [6000, 2500, 40], small=1500), 8, 10 ** 6, norm=1, cap=0)
    _record(ctx)


def test_score_modes(hgp, ctx):
    """a3's first tier: eta only (Delta cannot bind), packed with inter (tight Delta, uniform
    |e|), split (tight Delta, mixed c(e) too large to pack) — each against the oracle."""
    ctx.tier_counts(reset=True)
    # eta only: unbounded Delta
    _unfused_level(hgp, ctx, hgpgen.tiny(4), 16, hgpgen.UNBOUNDED)
    # packed with inter: SNN edges of equal size, Delta below in_mu(n) + max in_mu
    _unfused_level(hgp, ctx, hgpgen.snn(9, layers=3, rows=12, cols=12, fanout=20, window=7), 16, 80, cap=0)
    # split: mixed sizes and weights (gcd 1, sum c(e) / g shifted by the inter bits > 2^32)
    _unfused_level(hgp, ctx, _hubs(2, 3000, [60, 50], small=4000, smax=12, wmax=60), 8, 20)
    _record(ctx)


def test_fused_tiers(hgp, ctx):
    """The fused level-0 kernel: the sampled first tier, A, M (neighbourhoods of ~2800 through the
    sampling decision), B (a 6000-pin edge: neighbourhoods above M's 4096) and the hub tier (edges
    of 8700-9500 pins; weights up to 400 and a tight Delta: gcd and inter in the packed term)."""
    ctx.tier_counts(reset=True)
    cases = [(hgpgen.snn(8, layers=4, rows=40, cols=60, fanout=99, window=15, rewire=1.0), 256, 4096, 128),
             (hgpgen.snn(6, layers=3, rows=30, cols=30, fanout=60, window=11), 64, 4096, 128),
             (_hubs(3, 20000, [6000, 40], small=2000, wmax=1), 8, 10 ** 6, 65536),
             # hubs: b(n) > 8192 pin visits -> the key-partitioned hub tier (8 partitions per node)
             (_hubs(5, 20000, [9000, 40], small=2000, wmax=1), 8, 10 ** 6, 65536),
             (_hubs(6, 20000, [9500, 8700], small=2000, wmax=400), 8, 40, 65536)]
    for hg, omega, delta, smin in cases:
        with ctx.options(fused_sample_min=smin):
            cap = hgpgen.default_noise_cap(hg)
            g = gpu_build(hgp, ctx, hg)
            rg = ref.build_csr_hg(hg)
            rnb = ref.unique_neighbors(rg)
            # (the sampled first tier only runs from fused_sample_min nodes on)
            rr = ref.coarsen_level(rg, rnb, ref.params(omega, delta, 4, noise_seed=2, noise_cap=cap))
            m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
            gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
            cand = hgp.empty_cand(g.N, 4)
            nb, cg, cnb, _ = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap),
                                                cand, m, gam)
            assert_nbrs_equal(nb.to_host(), rnb, "fused nbrs")
            assert_cand_equal(hgp.cand_to_numpy(cand), rr["cand"])
            assert np.array_equal(m.cpu().numpy(), rr["match"])
            assert_csr_equal(cg.to_host(), rr["coarse"], "fused coarse")
            assert_nbrs_equal(cnb.to_host(), rr["coarse_nb"], "fused coarse nbrs")
            # the bench's form: N(n) left in the fused pool, N'(c) written over it in place
            cand2 = hgp.empty_cand(g.N, 4)
            _, cg2, cnb2, _ = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap),
                                                 cand2, m, gam, want_nbrs=False)
            assert_cand_equal(hgp.cand_to_numpy(cand2), rr["cand"])
            assert_csr_equal(cg2.to_host(), rr["coarse"], "fused coarse (in place)")
            assert_nbrs_equal(cnb2.to_host(), rr["coarse_nb"], "fused coarse nbrs (in place)")
            if hg.num_nodes == 20000 and omega == 8 and delta == 40:
                # hubs on the unfused list path instead (a2 list tiers, a3 list scoring)
                with ctx.options(no_hub=1):
                    cand3 = hgp.empty_cand(g.N, 4)
                    _, cg3, cnb3, _ = hgp.coarsen_level0(ctx, g, hgp.params(omega, delta, 4, noise_seed=2, noise_cap=cap),
                                                         cand3, m, gam, want_nbrs=False)
                    assert_cand_equal(hgp.cand_to_numpy(cand3), rr["cand"])
                    assert_nbrs_equal(cnb3.to_host(), rr["coarse_nb"], "unfused hubs, coarse nbrs")
    _record(ctx)


def test_pointer_jumping_tier(hgp, ctx):
    """A 3000-node path whose edge weights increase along it: node i targets i + 1, and every
    child's gain ss1 - ss0 stays > 0 (s_i > g_{i-1}, Eqs.9-10), so the best-child chain runs the
    whole path, far beyond the walk cap -> a4's pointer jumping."""
    ctx.tier_counts(reset=True)
    n = 3000
    off = np.arange(0, 2 * n + 1, 2, dtype=np.uint64)
    pins = np.stack([np.arange(n), np.arange(1, n + 1)], axis=1).reshape(-1).astype(np.uint32)
    hg = hgpgen.Hypergraph(n + 1, off, np.zeros(n, dtype=np.uint32), pins, np.arange(1, n + 1, dtype=np.uint32),
                           np.ones(n + 1, dtype=np.uint32))
    _unfused_level(hgp, ctx, hg, 2, 10, cap=0)
    _record(ctx)


def test_every_tier_was_exercised(hgp, ctx):
    from paper_2605_20497_b200.hgp import Ctx
    missing = [t for t in Ctx.TIERS if SEEN.get(t, 0) == 0]
    assert not missing, f"tiers never exercised: {missing}; counts {SEEN}"
