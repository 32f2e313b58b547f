"""World-size-2 gloo test of the multi-GPU host logic (paper_2605_20497_b200/shard.py): each rank
computes its node range's neighbours and candidates (here with the CPU oracle — the per-range
compute is the library's job on GPUs), the ranks all-gather them with allgather_v, and assemble()
must reproduce the unsharded level exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, bounds, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import hgpgen
    from oracle import ref
    from paper_2605_20497_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hg = hgpgen.tiny(3)
    g = ref.build_csr_hg(hg)
    lo, hi = bounds[rank], bounds[rank + 1]
    nb = ref.unique_neighbors(g, lo, hi)
    p = ref.params(16, 32, 4, noise_seed=2, noise_cap=1 << 22)
    cand = ref.score_pairs(g, nb, p)
    rows = np.stack([cand["id"][lo:hi].astype(np.int64), cand["score"][lo:hi].astype(np.int64)], axis=-1)
    t_rows = torch.from_numpy(rows.reshape(-1).copy())
    t_off = torch.from_numpy(nb.off.astype(np.int64))
    t_nbr = torch.from_numpy(nb.nbr.view(np.int32).copy())
    all_rows = shard.allgather_v(t_rows)
    all_off = shard.allgather_v(t_off)
    all_nbr = shard.allgather_v(t_nbr)
    c, off, nbr = shard.assemble(bounds, [r.view(-1, 4, 2) for r in all_rows], all_off, all_nbr)
    if rank == 0:
        out_q.put((c.numpy(), off.numpy(), nbr.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("bounds", [[0, 450, 1000], [0, 0, 1000], [0, 999, 1000]])
def test_gloo_world2_allgather_assemble_equals_unsharded(bounds):
    import hgpgen
    from oracle import ref
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, bounds, q)) for r in range(2)]
    for p in procs:
        p.start()
    c, off, nbr = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    hg = hgpgen.tiny(3)
    g = ref.build_csr_hg(hg)
    nb = ref.unique_neighbors(g)
    cand = ref.score_pairs(g, nb, ref.params(16, 32, 4, noise_seed=2, noise_cap=1 << 22))
    assert np.array_equal(c[..., 0].astype(np.uint32), cand["id"])
    assert np.array_equal(c[..., 1].astype(np.uint64), cand["score"])
    assert np.array_equal(off.astype(np.uint64), nb.off)
    assert np.array_equal(nbr.view(np.uint32), nb.nbr)


def _halo_worker(rank, world, port, out_q):
    """Rank `rank` of a gloo group: plans, packs and exchanges the halo of a level (shard.py) with
    oracle data, then checks that its segment view holds N(a) and N(b) of every coarse node it owns."""
    import sys
    sys.path.insert(0, ROOT)
    import hgpgen
    from oracle import ref
    from paper_2605_20497_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hg = hgpgen.tiny(5, num_nodes=600, num_edges=1500)
    g = ref.build_csr_hg(hg)
    nb_all = ref.unique_neighbors(g)
    rr = ref.coarsen_level(g, nb_all.copy(), ref.params(16, 32, 4, noise_seed=1, noise_cap=1 << 22))
    match = torch.from_numpy(rr["match"].view(np.int32).copy())
    N = g.N
    bounds = [(N * r) // world for r in range(world + 1)]
    lo, hi = bounds[rank], bounds[rank + 1]
    nb = ref.unique_neighbors(g, lo, hi)
    off = torch.from_numpy(nb.off.astype(np.int64))
    nbr = torch.from_numpy(nb.nbr.view(np.int32).copy())
    comm = shard.DistComm()
    b, dst = shard.halo_plan(match, bounds, rank)
    msgs = []
    for q in range(world):
        sel = b[dst == q]
        segs, ln = shard.pack_segments(off, nbr, lo, sel)
        msgs.append(shard.halo_message(sel, ln, segs))
    recv = comm.alltoall([msgs])[0]
    start, length, flat = shard.segment_view(N, lo, hi, off, nbr, recv)
    ok, checked = True, 0
    m = rr["match"]
    for a in range(lo, hi):
        p_ = int(m[a])
        if p_ != 0xFFFFFFFF and p_ < a:
            continue                      # a is not the min member: its coarse node is elsewhere
        for x in (a,) if p_ == 0xFFFFFFFF else (a, p_):
            s0, ln = int(start[x]), int(length[x])
            got = np.sort(flat[s0:s0 + ln].numpy().view(np.uint32))
            want = np.sort(nb_all.segment(x))
            ok &= np.array_equal(got, want)
            checked += 1
    out_q.put((rank, bool(ok), checked))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_halo_exchange():
    """X3 of the sharded level (shard.py) over a real gloo group of 2: every coarse node a rank owns
    sees both members' neighbour lists (its own, or its partner's from the other rank)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert sum(n for _, _, n in res) > 0


def test_edge_bounds_and_owner():
    from paper_2605_20497_b200 import shard
    off = torch.tensor([0, 5, 5, 9, 30, 31, 40], dtype=torch.int64)
    for world in (1, 2, 3, 8):
        b = shard.edge_bounds(off, world)
        assert b[0] == 0 and b[-1] == 6 and all(x <= y for x, y in zip(b, b[1:])) and len(b) == world + 1
    assert shard.owner_of([0, 3, 7, 10], torch.tensor([0, 2, 3, 6, 7, 9])).tolist() == [0, 0, 1, 1, 2, 2]
