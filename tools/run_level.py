"""Run the level-0 step (a1..a5) on a workload a few times — a short command for ncu / nsight.
Usage: python tools/run_level.py [--workload C2] [--steps 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import hgpgen
from paper_2605_20497_b200 import hgp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--hierarchy", action="store_true", help="run hgp_coarsen (all levels) instead of level 0")
    a = ap.parse_args()
    w = hgpgen.WORKLOADS[a.workload]
    hg = w.make(a.seed)
    omega = w.omega if w.omega > 0 else hgpgen.kway_omega(hg)
    ctx = hgp.Ctx(0)
    dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(hg, k))).cuda()
           for k in ("edge_off", "edge_nsrc", "pins", "edge_w", "node_w")}
    p = hgp.params(omega, w.delta, w.pi, noise_seed=a.seed, noise_cap=hgpgen.default_noise_cap(hg))
    N = hg.num_nodes
    cand = hgp.empty_cand(N, w.pi)
    m = torch.empty(N, dtype=torch.uint32, device="cuda")
    gam = torch.empty(N, dtype=torch.uint32, device="cuda")
    if a.hierarchy:
        for _ in range(a.steps):
            g = hgp.build_csr(ctx, N, dev["edge_off"], dev["edge_nsrc"], dev["pins"], dev["edge_w"], dev["node_w"])
            rho, cg, cnb, levels = hgp.coarsen(ctx, g, p)
            print(len(levels), "levels", flush=True)
            for x in (g, cg, cnb):
                x.free()
        torch.cuda.synchronize()
        return
    for _ in range(a.steps):
        g = hgp.build_csr(ctx, N, dev["edge_off"], dev["edge_nsrc"], dev["pins"], dev["edge_w"], dev["node_w"])
        nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, p, cand, m, gam)
        print(st, flush=True)
        for x in (g, nb, cg, cnb):
            x.free()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
