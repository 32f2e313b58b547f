import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, hgpgen
from oracle import ref
from paper_2605_20497_b200 import hgp
hg = hgpgen.vlsi(6, 20000, 20000, dmax=1024, in_cap=600)
cap = hgpgen.default_noise_cap(hg)
ctx = hgp.Ctx(0)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
g = hgp.build_csr(ctx, hg.num_nodes, dev(hg.edge_off), dev(hg.edge_nsrc), dev(hg.pins), dev(hg.edge_w), dev(hg.node_w))
cand = hgp.empty_cand(g.N, 4)
nb = hgp.neighbors_and_scores(ctx, g, hgp.params(64, 600, 4, noise_seed=2, noise_cap=cap), cand)
c = hgp.cand_to_numpy(cand)
rg = ref.build_csr_hg(hg); rnb = ref.unique_neighbors(rg)
rc = ref.score_pairs(rg, rnb, ref.params(64, 600, 4, noise_seed=2, noise_cap=cap))
bad = np.nonzero((c["id"] != rc["id"]).any(1) | (c["score"] != rc["score"]).any(1))[0]
print("bad nodes", len(bad), bad[:10])
for n in bad[:4]:
    K = rg.inc_off[n+1] - rg.inc_off[n]
    print(n, "K", K, "nbrs", rnb.off[n+1]-rnb.off[n], "gpu", c[n], "ref", rc[n])
