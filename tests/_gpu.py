"""Helpers for GPU-vs-oracle parity: run both paths on the same seeded input and compare.

Comparison rules: every integer array bit for bit, except the
contents of neighbour segments, which are sets (include/hgp.h): their offsets are
compared exactly and each segment is compared after sorting (flag bit included).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import ref

CSR_KEYS = ("edge_off", "edge_nsrc", "pins", "edge_w", "edge_mu", "node_w", "inc_off", "inc_nin", "inc", "in_mu")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_build(hgp, ctx, hg):
    return hgp.build_csr(ctx, hg.num_nodes, dev(hg.edge_off), dev(hg.edge_nsrc), dev(hg.pins), dev(hg.edge_w),
                         dev(hg.node_w))


def assert_csr_equal(h: dict, r: ref.Csr, what: str = "csr"):
    for k in CSR_KEYS:
        a, b = h[k], getattr(r, k)
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0] if a.shape == b.shape else []
            raise AssertionError(f"{what}.{k} differs: shapes {a.shape} vs {b.shape}; first bad {bad[:5]}; "
                                 f"gpu {a[bad[:5]] if len(bad) else a[:5]} oracle {b[bad[:5]] if len(bad) else b[:5]}")


def assert_nbrs_equal(h: dict, r: ref.Nbrs, what: str = "nbrs"):
    off, nbr = h["off"], h["nbr"]
    assert np.array_equal(off, r.off), f"{what}.off differs (first bad {np.nonzero(off != r.off)[0][:5]})"
    assert nbr.shape == r.nbr.shape, f"{what}.nbr size {nbr.shape} vs {r.nbr.shape}"
    # segments are sets: sort each one (flag bit included) — vectorised via a segment key
    seg = np.repeat(np.arange(len(off) - 1, dtype=np.int64), np.diff(off.astype(np.int64)))
    a = np.lexsort((nbr.astype(np.int64), seg))
    b = np.lexsort((r.nbr.astype(np.int64), seg))
    ga, gb = nbr[a], r.nbr[b]
    if not np.array_equal(ga, gb):
        bad = np.nonzero(ga != gb)[0][:5]
        raise AssertionError(f"{what}: segment sets differ at nodes {seg[a][bad]}: gpu {ga[bad]} oracle {gb[bad]}")


def assert_cand_equal(c_gpu: np.ndarray, c_ref: np.ndarray, lo: int = 0, hi: int | None = None):
    hi = c_ref.shape[0] if hi is None else hi
    a, b = c_gpu[lo:hi], c_ref[lo:hi]
    if not np.array_equal(a, b):
        bad = np.nonzero((a != b).any(axis=1))[0][:5]
        raise AssertionError(f"cand differs at nodes {bad + lo}: gpu {a[bad].tolist()} oracle {b[bad].tolist()}")
