"""GPU f2 (hgp_leftover_pairs) vs the oracle: the extra DP round on
random leftover instances (direct call), and whole levels / hierarchies with HGP_FLAG_LEFTOVER,
bit for bit."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import assert_csr_equal, assert_nbrs_equal, dev, gpu_build

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


def _cand_tensor(hgp, cand):
    raw = np.zeros((cand.shape[0], cand.shape[1], 2), dtype=np.uint64)
    raw[..., 0] = cand["id"].astype(np.uint64) | (cand["pad"].astype(np.uint64) << np.uint64(32))
    raw[..., 1] = cand["score"]
    return torch.from_numpy(raw.view(np.int64)).cuda()


@pytest.mark.parametrize("seed", range(12))
def test_leftover_round_matches_oracle(hgp, ctx, seed):
    rng = np.random.default_rng(100 + seed)
    N = int(rng.integers(2, 3000))
    w = rng.integers(1, 6, size=N).astype(np.uint32)
    mu = rng.integers(0, 5, size=N).astype(np.uint32)
    omega = int(rng.integers(2, 9))
    delta = ref.UNBOUNDED if seed % 3 == 0 else int(rng.integers(0, 8))
    cand = np.zeros((N, 2), dtype=ref.CAND_DTYPE)
    cand["id"] = ref.NONE
    has = rng.random(N) < 0.3                       # nodes with a regular candidate are not leftovers
    cand["id"][has, 0] = 0
    cand["score"][has, 0] = 1
    m0 = np.full(N, ref.NONE, dtype=np.uint32)
    rm, radd = ref.leftover_pairs(cand, w, mu, omega, delta, m0)
    mt = torch.from_numpy(m0.view(np.int32)).cuda()
    added = hgp.leftover_pairs(ctx, _cand_tensor(hgp, cand), N, 2, dev(w), dev(mu), omega, delta, mt)
    assert np.array_equal(mt.cpu().numpy().view(np.uint32), rm)
    assert added == radd


CASES = [
    ("C1-tight", lambda: hgpgen.tiny(5, num_nodes=300, num_edges=200, size_binom=4), 4, 8),
    ("vlsi-tight", lambda: hgpgen.vlsi(9, 400, 300, dmax=20, in_cap=12), 6, 14),
    ("C1", lambda: hgpgen.tiny(1), 16, 32),
]


@pytest.mark.parametrize("pi,noise", [(4, False), (2, True)])
@pytest.mark.parametrize("name,make,omega,delta", CASES, ids=[c[0] for c in CASES])
def test_level_and_hierarchy_with_leftover(hgp, ctx, name, make, omega, delta, pi, noise):
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    rg = ref.build_csr_hg(hg)
    cap = hgpgen.default_noise_cap(hg) if noise else 0
    p = hgp.params(omega, delta, pi, noise_seed=5, noise_cap=cap, flags=hgp.FLAG_LEFTOVER)
    rp = ref.params(omega, delta, pi, noise_seed=5, noise_cap=cap)
    # unfused level (a3 on N(n)) and the fused level-0 path
    nb = hgp.unique_neighbors(ctx, g)
    m = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    cg, cnb, _ = hgp.coarsen_level(ctx, g, nb, p, None, m, gam)
    rr = ref.coarsen_level(rg, ref.unique_neighbors(rg), rp, leftover=True)
    assert np.array_equal(m.cpu().numpy(), rr["match"])
    assert_csr_equal(cg.to_host(), rr["coarse"], "level with f2")
    m0 = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    g0 = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    _, cg0, cnb0, _ = hgp.coarsen_level0(ctx, g, p, None, m0, g0, want_nbrs=False)
    assert np.array_equal(m0.cpu().numpy(), rr["match"])
    assert_nbrs_equal(cnb0.to_host(), rr["coarse_nb"], "fused level with f2")
    # whole hierarchy
    rho, cl, cln, levels = hgp.coarsen(ctx, g, p)
    r = ref.coarsen(rg, rp, leftover=True)
    assert len(levels) == len(r["levels"]) and np.array_equal(rho.cpu().numpy(), r["rho"])
    assert_csr_equal(cl.to_host(), r["coarsest"], "coarsest with f2")
