"""GPU vs oracle at BASELINE.json's full sizes, in the launch configuration bench.py times
(hgp_build_csr + hgp_coarsen_level0 on the seeded workload):
  a1  the whole CSR, bit for bit (oracle a1 on the full input);
  a2/a3  N(n), flags and cand on sampled node ranges (oracle on those ranges; first and last
         nodes included);
  a4  the whole match (oracle DP on the GPU's full candidate array, and the oracle's own
      candidates on the sampled ranges agree with the GPU's);
  a5  gamma in full (from match by definition), size conservation, Omega/Delta of every coarse
      node, every coarse edge of a sample recomputed from its fine edge, coarse incidence
      consistency, and the coarse neighbour sets of sampled coarse nodes.
"""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import assert_csr_equal, gpu_build

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

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


def _seg(off, arr, i):
    return arr[int(off[i]):int(off[i + 1])]


@pytest.mark.parametrize("wl", ["C2", "C2r", "C3"])
def test_full_size_level_sampled_parity(hgp, ctx, wl):
    w = hgpgen.WORKLOADS[wl]
    hg = w.make(1)
    omega, delta, pi = w.omega, w.delta, w.pi
    cap = hgpgen.default_noise_cap(hg)
    N = hg.num_nodes
    # ---- GPU, exactly as bench.py's step
    g = gpu_build(hgp, ctx, hg)
    p = hgp.params(omega, delta, pi, noise_seed=1, noise_cap=cap)
    cand = hgp.empty_cand(N, pi)
    m = torch.empty(N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(N, dtype=torch.uint32, device="cuda")
    nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, p, cand, m, gam)
    gh = g.to_host()
    nbh = nb.to_host()
    ch = cg.to_host()
    cnbh = cnb.to_host()
    c_gpu = hgp.cand_to_numpy(cand)
    m_gpu = m.cpu().numpy()
    gam_gpu = gam.cpu().numpy()
    # ---- a1 in full
    rg = ref.build_csr_hg(hg)
    assert_csr_equal(gh, rg, f"{wl} a1")
    # ---- a2 + a3 on sampled ranges (the oracle's a3 flags only its own range's rows)
    rp = ref.params(omega, delta, pi, noise_seed=1, noise_cap=cap)
    ranges = [(0, 300), (N // 3, N // 3 + 300), (N // 2 + 17, N // 2 + 317), (N - 300, N)]
    for lo, hi in ranges:
        rnb = ref.unique_neighbors(rg, lo, hi)
        rc = ref.score_pairs(rg, rnb, rp)
        assert np.array_equal(c_gpu[lo:hi], rc[lo:hi]), f"{wl} cand differs in [{lo},{hi})"
        for n in range(lo, hi):
            a = np.sort(_seg(nbh["off"], nbh["nbr"], n))
            b = np.sort(rnb.segment(n))
            assert np.array_equal(a, b), f"{wl} N({n}) / flags differ"
    # ---- a4 in full: the oracle DP on the GPU's candidates
    rm, rper, _ = ref.match(c_gpu, pi)
    assert np.array_equal(m_gpu, rm), f"{wl} match differs"
    assert st["matched_per_round"] == [int(x) for x in rper]
    # ---- a5: gamma by definition (coarse ids by ascending min member)
    rep = (m_gpu == ref.NONE) | (np.arange(N, dtype=np.int64) < m_gpu.astype(np.int64))
    cid = np.cumsum(rep) - 1
    lo_member = np.where(m_gpu == ref.NONE, np.arange(N), np.minimum(np.arange(N), m_gpu.astype(np.int64)))
    assert np.array_equal(gam_gpu, cid[lo_member].astype(np.uint32))
    Nc = int(rep.sum())
    assert cg.N == Nc == st["Nc"]
    # sizes conserved, Omega / Delta per coarse node
    cw = np.bincount(gam_gpu, weights=hg.node_w.astype(np.float64), minlength=Nc)
    assert np.array_equal(ch["node_w"].astype(np.float64), cw)
    assert int(ch["node_w"].max()) <= omega
    if delta != hgpgen.UNBOUNDED:
        assert int(ch["in_mu"].max()) <= delta
    # coarse incidence consistent with coarse edges: sum |I(c)| = P', in-counts = dst pins
    Pc = int(ch["edge_off"][-1])
    assert int(ch["inc_off"][-1]) == Pc
    dst_cnt = np.zeros(Nc, dtype=np.int64)
    sizes = np.diff(ch["edge_off"].astype(np.int64))
    ebase = np.repeat(ch["edge_off"][:-1].astype(np.int64) + ch["edge_nsrc"].astype(np.int64), sizes)
    is_dst = np.arange(Pc) >= ebase
    np.add.at(dst_cnt, ch["pins"][is_dst].astype(np.int64), 1)
    assert np.array_equal(dst_cnt, ch["inc_nin"].astype(np.int64))
    # sampled coarse edges recomputed from their class: each kept fine edge maps to the coarse
    # edge of its representative; with no merges/drops the coarse id equals the fine id
    if st["merged_edges"] == 0 and st["dropped_edges"] == 0:
        rng = np.random.default_rng(5)
        for e in rng.choice(hg.num_edges, size=2000, replace=False):
            lo, s_, hi = int(gh["edge_off"][e]), int(gh["edge_off"][e]) + int(gh["edge_nsrc"][e]), int(gh["edge_off"][e + 1])
            D = sorted(set(int(x) for x in gam_gpu[gh["pins"][s_:hi]]))
            S = sorted(set(int(x) for x in gam_gpu[gh["pins"][lo:s_]]) - set(D))
            clo, cs = int(ch["edge_off"][e]), int(ch["edge_off"][e]) + int(ch["edge_nsrc"][e])
            chi = int(ch["edge_off"][e + 1])
            assert list(ch["pins"][clo:cs]) == S and list(ch["pins"][cs:chi]) == D, f"coarse edge {e}"
            assert ch["edge_w"][e] == gh["edge_w"][e] and ch["edge_mu"][e] == gh["edge_mu"][e]
    # sampled coarse neighbour sets: gamma(N(a) ∪ N(b)) minus OR-flagged minus self
    rng = np.random.default_rng(7)
    members = {}
    for c in rng.choice(Nc, size=200, replace=False):
        members[int(c)] = None
    first = np.full(Nc, -1, dtype=np.int64)
    order = np.arange(N)
    first[gam_gpu[::-1]] = order[::-1]          # min member per coarse node
    for c in members:
        a = int(first[c])
        b = int(m_gpu[a]) if m_gpu[a] != ref.NONE else None
        X, F = set(), set()
        for x in [a] + ([b] if b is not None else []):
            for v in _seg(nbh["off"], nbh["nbr"], x):
                gv = int(gam_gpu[int(v) & 0x7FFFFFFF])
                X.add(gv)
                if int(v) & ref.PURGE:
                    F.add(gv)
        want = sorted(X - F - {c})
        assert sorted(int(x) for x in _seg(cnbh["off"], cnbh["nbr"], c)) == want, f"coarse N({c})"
