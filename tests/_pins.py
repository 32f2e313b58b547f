"""Independent checks ("pins") used to validate the oracle and the CUDA path.

Nothing here calls oracle/ or the product: these are the paper's definitions
evaluated by *different* means (dense incidence-matrix products instead of the
histogram traversal, exhaustive enumeration instead of the DP, explicit set
unions instead of the inline counter), plus the level's invariants.
"""
from __future__ import annotations

import itertools

import numpy as np

NONE = 0xFFFFFFFF
PURGE = 0x80000000
M64 = (1 << 64) - 1


# ----------------------------------------------------------------------------- hypergraph views
def edges_of(edge_off, edge_nsrc, pins):
    """List of (src set, dst set) per edge."""
    out = []
    for e in range(len(edge_nsrc)):
        lo, hi = int(edge_off[e]), int(edge_off[e + 1])
        s = lo + int(edge_nsrc[e])
        out.append((set(int(x) for x in pins[lo:s]), set(int(x) for x in pins[s:hi])))
    return out


def incidence_bruteforce(N, edges):
    """in(n), out(n) by scanning every edge for every node."""
    ins = [[e for e, (S, D) in enumerate(edges) if n in D] for n in range(N)]
    outs = [[e for e, (S, D) in enumerate(edges) if n in S] for n in range(N)]
    return ins, outs


# ----------------------------------------------------------------------------- metrics (Eq.1, Eq.2, Eq.16)
def connectivity(edges, w, rho):
    """Conn_G(rho) = sum_e omega(e) (lambda(e) - 1) (Eq.1)."""
    return sum(int(w[e]) * (len({int(rho[n]) for n in S | D}) - 1) for e, (S, D) in enumerate(edges))


def cut_net(edges, w, rho):
    """sum_e omega(e) [lambda(e) > 1] (Eq.16)."""
    return sum(int(w[e]) for e, (S, D) in enumerate(edges) if len({int(rho[n]) for n in S | D}) > 1)


def coarsening_score(edges, w, gamma):
    """Score_G(gamma) = sum_e omega(e) (|e| - |gamma(e)|) (Eq.2)."""
    return sum(int(w[e]) * (len(S | D) - len({int(gamma[n]) for n in S | D})) for e, (S, D) in enumerate(edges))


def inbound_counts(edges, mu, rho, nparts):
    """Per partition: sum of mu(e) over edges with a destination in the partition (reading #12)."""
    cnt = [0] * nparts
    for e, (S, D) in enumerate(edges):
        for p in {int(rho[n]) for n in D}:
            cnt[p] += int(mu[e])
    return cnt


# ----------------------------------------------------------------------------- a3 by matrix products
def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def noise(n, m, seed, cap):
    if cap == 0:
        return 0
    key = (min(n, m) << 32) | max(n, m)
    return (splitmix64(key ^ splitmix64(seed)) * (cap + 1)) >> 64


def score_bruteforce(N, edge_off, edge_nsrc, pins, edge_w, edge_mu, node_w, omega, delta, pi,
                     norm=0, seed=0, cap=0, unbounded=M64, live=None):
    """All-pairs eta / inter via dense incidence-matrix products (exact in float64: every
    partial sum < 2^53 for the sizes used here), then validity, flags and top-Pi by
    exhaustive sort.  eta(n,m) = sum_{e in I(n) cap I(m)} c(e) (Eq.5),
    inter(n,m) = sum_{e : n,m in dst(e)} mu(e).  ``live[n]`` optionally
    restricts n's bins (purge bits already set)."""
    E = len(edge_nsrc)
    sizes = np.diff(edge_off.astype(np.int64))
    c = (edge_w.astype(np.int64) << 24) if norm else ((edge_w.astype(np.int64) << 24) // np.maximum(sizes, 1))
    Mc = np.zeros((N, E))
    M1 = np.zeros((N, E))
    Md = np.zeros((N, E))
    Mdmu = np.zeros((N, E))
    for e in range(E):
        lo, hi = int(edge_off[e]), int(edge_off[e + 1])
        s = lo + int(edge_nsrc[e])
        for j in range(lo, hi):
            n = int(pins[j])
            Mc[n, e] = float(c[e])
            M1[n, e] = 1.0
            if j >= s:
                Md[n, e] = 1.0
                Mdmu[n, e] = float(edge_mu[e])
    assert float(c.sum()) * 2 < 2 ** 53
    eta = np.rint(Mc @ M1.T).astype(np.int64)
    inter = np.rint(Mdmu @ Md.T).astype(np.int64)
    adj = (M1 @ M1.T) > 0
    np.fill_diagonal(adj, False)
    in_mu = np.rint(Mdmu.sum(axis=1)).astype(np.int64)
    cand = []
    flagged = set()
    for n in range(N):
        vals = []
        for m in np.nonzero(adj[n])[0]:
            m = int(m)
            if live is not None and m not in live[n]:
                continue
            ok = int(node_w[n]) + int(node_w[m]) <= omega and (
                delta == unbounded or int(in_mu[n]) + int(in_mu[m]) - int(inter[n, m]) <= delta)
            if not ok:
                flagged.add((n, m))
                continue
            vals.append((int(eta[n, m]) + noise(n, m, seed, cap), m))
        vals.sort(key=lambda t: (-t[0], -t[1]))
        cand.append([(m, s) for s, m in vals[:pi]])
    return {"eta": eta, "inter": inter, "adj": adj, "in_mu": in_mu, "cand": cand, "flagged": flagged}


# ----------------------------------------------------------------------------- a4 by enumeration
def max_matching_bruteforce(nodes, edges_w):
    """Maximum total weight over all matchings of a small graph (exhaustive). edges_w: {(u,v): w}."""
    items = sorted(edges_w.items())
    best = 0
    # branch over edges in order: take or skip
    def rec(i, used, total):
        nonlocal best
        if i == len(items):
            best = max(best, total)
            return
        (u, v), w = items[i]
        rec(i + 1, used, total)
        if u not in used and v not in used:
            rec(i + 1, used | {u, v}, total + w)
    rec(0, frozenset(), 0)
    return best


def proposal_components(t):
    """Weakly connected components of the proposal graph n -> t(n) (t(n) = NONE: no edge)."""
    N = len(t)
    parent = list(range(N))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    for n in range(N):
        if t[n] != NONE:
            a, b = find(n), find(t[n])
            if a != b:
                parent[a] = b
    comps = {}
    for n in range(N):
        comps.setdefault(find(n), []).append(n)
    return list(comps.values())


def round_graph(cand, i, matched):
    """Round-i proposal graph with earlier-matched nodes removed."""
    N = cand.shape[0]
    t = [NONE] * N
    s = [0] * N
    for n in range(N):
        cid = int(cand[n, i]["id"])
        if not matched[n] and cid != NONE and not matched[cid]:
            t[n] = cid
            s[n] = int(cand[n, i]["score"])
    return t, s


def has_only_two_cycles(t):
    N = len(t)
    color = [0] * N
    for start in range(N):
        path = []
        x = start
        while x != NONE and color[x] == 0:
            color[x] = 1
            path.append(x)
            x = t[x]
        if x != NONE and color[x] == 1:       # new cycle found on this path
            cyc = path[path.index(x):]
            if len(cyc) != 2:
                return False
        for y in path:
            color[y] = 2
    return True
