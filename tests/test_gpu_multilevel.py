"""GPU multi-level driver (hgp_coarsen) vs the oracle driver
(oracle/ref.py coarsen): same number of levels, same per-level counts and matched pairs, the same
composed map rho = gamma^L o ... o gamma^1 and the same coarsest CSR / neighbour lists, bit for bit
(neighbour segments as sets)."""
import numpy as np
import pytest

import hgpgen
from oracle import ref
from tests._gpu import assert_csr_equal, assert_nbrs_equal, gpu_build

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = [
    ("C1", lambda: hgpgen.tiny(1), 16, 32),
    ("C1-w3", lambda: hgpgen.tiny(2, wmax_n=3), 16, 32),
    ("snn-small", lambda: hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30, window=9, rewire=0.1), 64, 256),
    ("vlsi-small", lambda: hgpgen.vlsi(6, 5000, 5000, dmax=200, in_cap=100), 32, 128),
    ("kway", lambda: hgpgen.vlsi(7, 2000, 2000, dmax=60, in_cap=10 ** 6), 1030, ref.UNBOUNDED),
]


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


@pytest.mark.parametrize("name,make,omega,delta", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("cap", [0, 1 << 22])
def test_multilevel_matches_oracle(hgp, ctx, name, make, omega, delta, cap):
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    rho, cg, cnb, levels = hgp.coarsen(ctx, g, hgp.params(omega, delta, 4, noise_seed=3, noise_cap=cap))
    r = ref.coarsen(ref.build_csr_hg(hg), ref.params(omega, delta, 4, noise_seed=3, noise_cap=cap))
    assert len(levels) == len(r["levels"])
    for a, b in zip(levels, r["levels"]):
        assert (a["N"], a["E"], a["P"], a["Nc"], a["Ec"], a["Pc"]) == (b["N"], b["E"], b["P"], b["Nc"], b["Ec"], b["Pc"])
        assert a["matched_per_round"] == b["matched_per_round"]
    assert np.array_equal(rho.cpu().numpy(), r["rho"])
    assert_csr_equal(cg.to_host(), r["coarsest"], "coarsest")
    assert_nbrs_equal(cnb.to_host(), r["coarsest_nb"], "coarsest nbrs")
    g.free(); cg.free(); cnb.free()


def test_multilevel_max_levels_and_args(hgp, ctx):
    hg = hgpgen.tiny(4)
    g = gpu_build(hgp, ctx, hg)
    rho, cg, cnb, levels = hgp.coarsen(ctx, g, hgp.params(16, 32, 4), max_levels=1)
    r = ref.coarsen(ref.build_csr_hg(hg), ref.params(16, 32, 4), max_levels=1)
    assert len(levels) == 1 and np.array_equal(rho.cpu().numpy(), r["rho"])
    assert_csr_equal(cg.to_host(), r["coarsest"], "coarsest")
    cg.free(); cnb.free()
    with pytest.raises(hgp.HgpError):
        hgp.coarsen(ctx, g, hgp.params(16, 32, 4), max_levels=0)
    g.free()
