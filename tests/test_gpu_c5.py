"""C5 (BASELINE.json config 5: the billion-pin SNN, 10^7 neurons, 10^9 pins) on ONE B200 — the
only configuration whose neighbour lists exceed 2^32 entries (64-bit neighbour offsets, the fused
kernel's 2^34-entry pool cap). In bench.py's launch configuration (hgp_coarsen_level0, N(n)
consumed by a5 in place):
  a1      sampled slices of the CSR equal the oracle's full-size a1 (incidence offsets and lists of
          sampled nodes, pins of sampled edges);
  a2+a3   cand of sampled node ranges equals the oracle's a2 + a3 on those ranges;
  a4      the whole match equals the oracle DP on the GPU's candidates;
  a5      invariants at full size: N' = N - pairs, sizes conserved and <= Omega, in_mu' <= Delta,
          coarse incidence consistent with the coarse edges.
"""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import gpu_build

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


def test_c5_billion_pins_one_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_20497_b200 import hgp
    ctx = hgp.Ctx(0)
    w = hgpgen.WORKLOADS["C5"]
    hg = w.make(1)
    N, P = hg.num_nodes, hg.num_pins
    assert P >= 10 ** 9
    cap = hgpgen.default_noise_cap(hg)
    g = gpu_build(hgp, ctx, hg)
    p = hgp.params(w.omega, w.delta, w.pi, noise_seed=1, noise_cap=cap)
    cand = hgp.empty_cand(N, w.pi)
    m = torch.empty(N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(N, dtype=torch.uint32, device="cuda")
    _, cg, cnb, st = hgp.coarsen_level0(ctx, g, p, cand, m, gam, want_nbrs=False)
    assert st["V"] > 2 ** 32, st["V"]                      # the 64-bit neighbour offsets are exercised
    c_gpu = hgp.cand_to_numpy(cand)
    m_gpu = m.cpu().numpy()
    gt = g.tensors()
    # ---- oracle a1 in full; sampled comparisons of the CSR
    rg = ref.build_csr_hg(hg)
    rng = np.random.default_rng(5)
    nodes = np.unique(np.concatenate([[0, N - 1], rng.integers(0, N, size=200)]))
    inc_off = gt["inc_off"].cpu().numpy()
    assert np.array_equal(inc_off[nodes], rg.inc_off[nodes]) and inc_off[-1] == rg.inc_off[-1]
    for n in nodes[:50]:
        a, b = int(rg.inc_off[n]), int(rg.inc_off[n + 1])
        assert np.array_equal(gt["inc"][a:b].cpu().numpy(), rg.inc[a:b])
    for e in rng.integers(0, hg.num_edges, size=50):
        a, b = int(rg.edge_off[e]), int(rg.edge_off[e + 1])
        assert np.array_equal(gt["pins"][a:b].cpu().numpy(), rg.pins[a:b])
    # ---- a2 + a3 on sampled ranges
    rp = ref.params(w.omega, w.delta, w.pi, noise_seed=1, noise_cap=cap)
    for lo, hi in [(0, 200), (N // 2, N // 2 + 200), (N - 200, N)]:
        rc = ref.score_pairs(rg, ref.unique_neighbors(rg, lo, hi), rp)
        assert np.array_equal(c_gpu[lo:hi], rc[lo:hi]), f"C5 cand differs in [{lo},{hi})"
    # ---- a4 in full: the oracle DP on the GPU's candidates
    rm, rper, _ = ref.match(c_gpu, w.pi)
    assert np.array_equal(m_gpu, rm)
    # ---- a5 invariants at full size
    pairs = int((m_gpu != ref.NONE).sum()) // 2
    assert cg.N == N - pairs
    ch = {k: v.cpu().numpy() for k, v in cg.tensors().items() if k in ("node_w", "in_mu", "inc_off", "edge_off")}
    assert int(ch["node_w"].astype(np.int64).sum()) == int(hg.node_w.astype(np.int64).sum())
    assert ch["node_w"].max() <= w.omega and ch["in_mu"].max() <= w.delta
    assert int(ch["inc_off"][-1]) == int(ch["edge_off"][-1]) == cg.P
