"""Multi-GPU sharding logic on one GPU: W logical ranks run their node ranges one after the other
and are assembled exactly as the NCCL all-gathers would (shard.level0_loopback); the result must be
bit-identical to the single-GPU level."""
import numpy as np
import pytest

import hgpgen
from tests._gpu import assert_csr_equal, assert_nbrs_equal, gpu_build

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hgp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_20497_b200 import hgp as h
    h.lib()
    return h


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name,make,omega,delta", [
    ("snn", lambda: hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30, window=9, rewire=0.1), 16, 256),
    ("vlsi", lambda: hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600), 64, 600),
])
def test_loopback_shards_equal_single_gpu(hgp, world, name, make, omega, delta):
    from paper_2605_20497_b200 import shard
    ctx = hgp.Ctx(0)
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    p = hgp.params(omega, delta, 4, noise_seed=3, noise_cap=hgpgen.default_noise_cap(hg))
    N = g.N
    outs = []
    for mode in ("single", "sharded"):
        cand = hgp.empty_cand(N, 4)
        m = torch.empty(N, dtype=torch.uint32, device="cuda")
        gam = torch.empty(N, dtype=torch.uint32, device="cuda")
        if mode == "single":
            nb, cg, cnb, _ = hgp.coarsen_level0(ctx, g, p, cand, m, gam)
        else:
            nb, cg, cnb, bounds = shard.level0_loopback(ctx, g, p, cand, m, gam, world)
            assert bounds[0] == 0 and bounds[-1] == N and all(a <= b for a, b in zip(bounds, bounds[1:]))
        outs.append((cand.cpu().numpy(), m.cpu().numpy(), gam.cpu().numpy(), nb.to_host(), cg, cnb.to_host()))
    (c0, m0, g0, nb0, cg0, cnb0), (c1, m1, g1, nb1, cg1, cnb1) = outs
    assert np.array_equal(c0, c1) and np.array_equal(m0, m1) and np.array_equal(g0, g1)
    for k in ("off",):
        assert np.array_equal(nb0[k], nb1[k]) and np.array_equal(cnb0[k], cnb1[k])
    seg = lambda h: np.repeat(np.arange(len(h["off"]) - 1), np.diff(h["off"].astype(np.int64)))
    for a, b in ((nb0, nb1), (cnb0, cnb1)):
        ia, ib = np.lexsort((a["nbr"], seg(a))), np.lexsort((b["nbr"], seg(b)))
        assert np.array_equal(a["nbr"][ia], b["nbr"][ib])
    h0, h1 = cg0.to_host(), cg1.to_host()
    for k in h0:
        assert np.array_equal(h0[k], h1[k]), k


def test_shard_bounds_balance(hgp):
    ctx = hgp.Ctx(0)
    hg = hgpgen.vlsi(9, 50000, 50000, dmax=1024, in_cap=1000)
    g = gpu_build(hgp, ctx, hg)
    b = hgp.shard_bounds(ctx, g, 8)
    h = g.to_host()
    sizes = np.diff(h["edge_off"].astype(np.int64))
    inc = h["inc"].astype(np.int64)
    work = np.add.reduceat(sizes[inc], h["inc_off"][:-1].astype(np.int64)) if len(inc) else np.zeros(g.N)
    work = np.where(np.diff(h["inc_off"].astype(np.int64)) > 0, work, 0) + 1
    pre = np.concatenate([[0], np.cumsum(work)])
    shares = [pre[b[r + 1]] - pre[b[r]] for r in range(8)]
    assert b[0] == 0 and b[-1] == g.N
    assert max(shares) <= pre[-1] / 8 + work.max() + 1
