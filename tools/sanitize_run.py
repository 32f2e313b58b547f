"""Small end-to-end run of every product entry point for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): a1, fused level 0 (and the unfused path), a3/a4/a5 on the next level, the
multi-level driver with f2, and the f1/f3/f4 calls, on C1 and an SNN sample.
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import hgpgen
from paper_2605_20497_b200 import hgp


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(hg, omega, delta, unfused):
    ctx = hgp.Ctx(0, allocator="builtin")   # library arrays via cudaMallocAsync (exact sizes for memcheck)
    ctx.set_option("unfused", int(unfused))
    g = hgp.build_csr(ctx, hg.num_nodes, dev(hg.edge_off), dev(hg.edge_nsrc), dev(hg.pins), dev(hg.edge_w),
                      dev(hg.node_w))
    N = g.N
    p = hgp.params(omega, delta, 4, noise_seed=3, noise_cap=hgpgen.default_noise_cap(hg), flags=hgp.FLAG_LEFTOVER)
    cand = hgp.empty_cand(N, 4)
    m = torch.empty(N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(N, dtype=torch.uint32, device="cuda")
    nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, p, cand, m, gam)
    m2 = torch.empty(cg.N, dtype=torch.uint32, device="cuda")
    g2 = torch.empty(cg.N, dtype=torch.uint32, device="cuda")
    c2, cn2, _ = hgp.coarsen_level(ctx, cg, cnb, p, None, m2, g2)
    rho, cl, cln, levels = hgp.coarsen(ctx, g, p)
    q = hgp.partition_metrics(ctx, g, rho, cl.N, omega, delta)
    pins = hgp.pins_matrix(ctx, g, rho, cl.N)
    d, gn = hgp.propose_moves(ctx, g, rho, cl.N, omega, True, pins=pins)
    movers = torch.nonzero(d.view(torch.int32) != -1).flatten()
    seq = movers[torch.argsort(-gn[movers], stable=True)].to(torch.int32).contiguous()
    gs = hgp.in_sequence_gains(ctx, g, rho, cl.N, seq, d, pins=pins)
    v = hgp.sequence_violations(ctx, g, rho, cl.N, seq, d, omega, delta)
    k, best = hgp.best_prefix(ctx, gs, v)
    torch.cuda.synchronize()
    print(hg.name, "unfused" if unfused else "fused", "levels", len(levels), "conn", q["connectivity"], "k", k, flush=True)


def hubs(seed=7, N=12000, big=(9000, 40), small=1000, smax=30):
    """Edges of 9000 pins among small ones: fused-level hub nodes (b > 8192, hub.cu) and a5 coarse
    hubs (|N(a)| + |N(b)| > 16384, the key-partitioned coarse tier)."""
    rng = np.random.default_rng(seed)
    sizes = list(big) + [int(x) for x in rng.integers(2, smax, size=small)]
    pins, nsrc, off = [], [], [0]
    for s in sizes:
        pins.extend(rng.choice(N, size=s, replace=False).tolist())
        nsrc.append(int(rng.integers(0, 3)) if s > 2 else 1)
        off.append(len(pins))
    return hgpgen.Hypergraph(N, np.array(off, dtype=np.uint64), np.array(nsrc, dtype=np.uint32),
                             np.array(pins, dtype=np.uint32), rng.integers(1, 9, size=len(sizes)).astype(np.uint32),
                             np.ones(N, dtype=np.uint32), name="hubs")


if __name__ == "__main__":
    for unfused in (False, True):
        run(hubs(), 8, 10 ** 6, unfused)
        run(hgpgen.tiny(1), 16, 32, unfused)
        run(hgpgen.snn(2, layers=3, rows=20, cols=20, fanout=30, window=7, rewire=0.1), 64, 256, unfused)
        run(hgpgen.vlsi(3, 4000, 4000, dmax=300, in_cap=64), 32, 128, unfused)
    print("sanitize run ok")
