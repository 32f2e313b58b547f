"""Full-size oracle digests: run the CPU ORACLE (oracle/ only — no product code) on one whole
BASELINE workload and store SHA-256 digests of every output of the level in tests/golden/.

    python tools/golden_full.py --workload C2 --seed 1        # ~15 min on one core

Level = a1 (hgp_ref_build_csr) -> a2 (hgp_ref_unique_neighbors) -> a3 -> a4 -> a5
(hgp_ref_coarsen_level), parameters exactly as bench.py's step (Omega, Delta, Pi of the workload,
noise seed = the workload seed, noise cap = hgpgen.default_noise_cap).  Neighbour segments are
sets (DESIGN reading #15), so their digest is taken over each segment sorted by its raw u32
entries (flag bit included) — the same canonical form tests/test_gpu_golden.py builds from the
GPU's output.  The oracle's wall time per step is recorded too (the full-size CPU baseline,
one thread).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hgpgen  # noqa: E402
from oracle import ref  # noqa: E402

CSR_KEYS = ("edge_off", "edge_nsrc", "pins", "edge_w", "edge_mu", "node_w", "inc_off", "inc_nin", "inc", "in_mu")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def canonical_nbr(off: np.ndarray, nbr: np.ndarray) -> np.ndarray:
    """Each segment sorted by raw u32 value (flag bit included)."""
    out = nbr.copy()
    for i in range(len(off) - 1):
        lo, hi = int(off[i]), int(off[i + 1])
        if hi - lo > 1:
            out[lo:hi].sort()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    w = hgpgen.WORKLOADS[a.workload]
    hg = w.make(a.seed)
    omega = w.omega if w.omega > 0 else hgpgen.kway_omega(hg, w.extra.get("kway", 2))
    cap = hgpgen.default_noise_cap(hg) if w.noise else 0
    t = {}
    t0 = time.perf_counter()
    g = ref.build_csr_hg(hg)
    t["a1"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    nb = ref.unique_neighbors(g)
    t["a2"] = time.perf_counter() - t0
    p = ref.params(omega, w.delta, w.pi, noise_seed=a.seed, noise_cap=cap)
    t0 = time.perf_counter()
    cand = ref.score_pairs(g, nb, p)
    t["a3"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    m, per, _ = ref.match(cand, w.pi)
    t["a4"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    gamma, cg, cnb = ref.contract(g, nb, m)
    t["a5"] = time.perf_counter() - t0
    total = sum(t.values())
    d = {
        "_doc": "SHA-256 digests of the CPU oracle's level on a full BASELINE workload, written by "
                "tools/golden_full.py (oracle/ only). Neighbour digests: each segment sorted by raw u32 "
                "(flag bit included). Compared with the GPU by tests/test_gpu_golden.py.",
        "workload": w.name, "key": a.workload, "seed": a.seed, "omega": omega,
        "delta": "inf" if w.delta == ref.UNBOUNDED else w.delta, "pi": w.pi, "noise_cap": cap,
        "N": g.N, "E": g.E, "P": g.P, "V": int(nb.nbr.shape[0]), "Nc": cg.N, "Ec": cg.E, "Pc": cg.P,
        "Vc": int(cnb.nbr.shape[0]), "matched_per_round": [int(x) for x in per],
        "purged": int(np.count_nonzero(nb.nbr & ref.PURGE)),
        "sha256": {
            "csr": {k: sha(getattr(g, k)) for k in CSR_KEYS},
            "nb_off": sha(nb.off), "nb_nbr_sorted": sha(canonical_nbr(nb.off, nb.nbr)),
            "cand": sha(cand), "match": sha(m), "gamma": sha(gamma),
            "coarse": {k: sha(getattr(cg, k)) for k in CSR_KEYS},
            "coarse_nb_off": sha(cnb.off), "coarse_nb_nbr_sorted": sha(canonical_nbr(cnb.off, cnb.nbr)),
        },
        "oracle_seconds": {k: round(v, 2) for k, v in t.items()} | {"total": round(total, 2)},
        "oracle_pins_per_s": g.P / total,
        "oracle_host": {"cores_used": 1, "cpu": platform.processor() or platform.machine(),
                        "host_cores": os.cpu_count()},
    }
    out = os.path.join(ROOT, "tests", "golden", f"{a.workload}_s{a.seed}.json")
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps({k: d[k] for k in ("workload", "N", "P", "V", "Nc", "Ec", "oracle_seconds")}))


if __name__ == "__main__":
    main()
