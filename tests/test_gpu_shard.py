"""Multi-GPU schedule of the level and of the driver (paper_2605_20497_b200/shard.py)
on one GPU: W logical ranks (LoopbackComm, W = 2, 3, 8) and a real torch.distributed NCCL group
of one rank (DistComm), each against the single-GPU hgp_coarsen — bit for bit: levels, rho, the
coarsest CSR, and the coarsest neighbour lists assembled from the ranks' shards (compared as sets
per segment, reading #15)."""
import os
import socket

import numpy as np
import pytest

import hgpgen
from tests._gpu import assert_csr_equal, gpu_build

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hgp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_20497_b200 import hgp as h
    h.lib()
    return h


CASES = [
    ("snn", lambda: hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30, window=9, rewire=0.1), 16, 256, 0),
    ("vlsi", lambda: hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600), 64, 600, 0),
    ("C1-f2", lambda: hgpgen.tiny(1), 16, 32, 1),
]


def _sets(off, nbr):
    seg = np.repeat(np.arange(len(off) - 1), np.diff(off.astype(np.int64)))
    i = np.lexsort((nbr.astype(np.int64), seg))
    return nbr[i]


def _single(hgp, ctx, g, p):
    rho, cl, cln, levels = hgp.coarsen(ctx, g, p)
    return rho.cpu().numpy(), cl.to_host(), cln.to_host(), [l["Nc"] for l in levels]


def _check_sharded(hgp, ctx, g, p, comm, want):
    from paper_2605_20497_b200 import shard
    rho, levels, cl, states = shard.coarsen_sharded(ctx, g, p, comm)
    w_rho, w_cl, w_cln, w_nc = want
    assert [l.Nc for l in levels] == w_nc
    assert np.array_equal(rho.cpu().numpy(), w_rho)
    h = cl.to_host()
    for k in w_cl:
        assert np.array_equal(h[k], w_cl[k]), k
    # the coarsest neighbour lists: the ranks' contiguous coarse ranges, in rank order
    states = sorted(states, key=lambda s: s.r)
    assert states[0].lo == 0 and states[-1].hi == cl.N
    offs, nbrs = [], []
    for s in states:
        t = s.nb.to_host()
        offs.append(t["off"])
        nbrs.append(t["nbr"])
    base, off = 0, [np.uint64(0)]
    for o in offs:
        off.extend((o[1:] + base).tolist())
        base += int(o[-1])
    off = np.array(off, dtype=np.uint64)
    nbr = np.concatenate(nbrs) if nbrs else np.zeros(0, np.uint32)
    assert np.array_equal(off, w_cln["off"])
    assert np.array_equal(_sets(off, nbr), _sets(w_cln["off"], w_cln["nbr"]))
    return levels


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name,make,omega,delta,f2", CASES, ids=[c[0] for c in CASES])
def test_loopback_shards_equal_single_gpu(hgp, world, name, make, omega, delta, f2):
    from paper_2605_20497_b200 import shard
    ctx = hgp.Ctx(0)
    hg = make()
    g = gpu_build(hgp, ctx, hg)
    p = hgp.params(omega, delta, 4, noise_seed=3, noise_cap=hgpgen.default_noise_cap(hg),
                   flags=hgp.FLAG_LEFTOVER if f2 else 0)
    want = _single(hgp, ctx, g, p)
    levels = _check_sharded(hgp, ctx, g, p, shard.LoopbackComm(world), want)
    assert all(set(l.ms) >= {"a2a3", "X1", "a4", "X2", "X3"} for l in levels)


def test_nccl_group_of_one_equals_single_gpu(hgp):
    """shard.coarsen_sharded through a real torch.distributed NCCL process group (DistComm: the
    all-gathers and the batched send/recv halo exchange run through NCCL)."""
    import torch.distributed as dist
    from paper_2605_20497_b200 import shard
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ctx = hgp.Ctx(0)
        hg = hgpgen.snn(5, layers=4, rows=20, cols=20, fanout=30, window=9, rewire=0.1)
        g = gpu_build(hgp, ctx, hg)
        p = hgp.params(16, 256, 4, noise_seed=3, noise_cap=hgpgen.default_noise_cap(hg))
        _check_sharded(hgp, ctx, g, p, shard.DistComm(), _single(hgp, ctx, g, p))
    finally:
        dist.destroy_process_group()


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
