"""Per-kernel device time of the whole multi-level hierarchy (hgp_coarsen) on a workload:
one warm-up run, then one profiled run. Usage: python tools/hier_profile.py [--workload C2]"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import hgpgen
from paper_2605_20497_b200 import hgp

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
a = ap.parse_args()
w = hgpgen.WORKLOADS[a.workload]
hg = w.make(1)
omega = w.omega if w.omega > 0 else hgpgen.kway_omega(hg)
ctx = hgp.Ctx(0)
dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(hg, k))).cuda() for k in ("edge_off", "edge_nsrc", "pins", "edge_w", "node_w")}
p = hgp.params(omega, w.delta, w.pi, noise_seed=1, noise_cap=hgpgen.default_noise_cap(hg))
for it in range(2):
    g = hgp.build_csr(ctx, hg.num_nodes, dev["edge_off"], dev["edge_nsrc"], dev["pins"], dev["edge_w"], dev["node_w"])
    torch.cuda.synchronize()
    if it == 1:
        ctx.profile_begin("")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    rho, cg, cnb, levels = hgp.coarsen(ctx, g, p)
    ev1.record()
    torch.cuda.synchronize()
    if it == 1:
        ctx.profile_end()
        rep = ctx.profile_report()
        tot = sum(v[0] for v in rep.values())
        print(f"hierarchy {ev0.elapsed_time(ev1):.1f} ms (profiled run), {len(levels)} levels, kernel sum {tot:.1f} ms")
        for k, (ms, n) in sorted(rep.items(), key=lambda kv: -kv[1][0])[:30]:
            print(f"  {k:28s} {ms:9.3f} ms  {n:6d} launches")
    for x in (g, cg, cnb):
        x.free()
