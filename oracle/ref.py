"""ctypes binding of the CPU ORACLE (oracle/libhgp_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs — never by the product
package.  Host numpy arrays in, host numpy arrays out.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

NONE = 0xFFFFFFFF
UNBOUNDED = (1 << 64) - 1
PURGE = 0x80000000
FP_SHIFT = 24

u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)


class CInput(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_uint32), ("num_edges", ctypes.c_uint32),
                ("edge_off", u64p), ("edge_nsrc", u32p), ("pins", u32p),
                ("edge_w", u32p), ("node_w", u32p)]


class CCsr(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint32), ("E", ctypes.c_uint32), ("P", ctypes.c_uint64),
                ("edge_off", u64p), ("edge_nsrc", u32p), ("pins", u32p), ("edge_w", u32p),
                ("edge_mu", u32p), ("node_w", u32p), ("inc_off", u64p), ("inc_nin", u32p),
                ("inc", u32p), ("in_mu", u32p)]


class CNbrs(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_uint32), ("hi", ctypes.c_uint32), ("V", ctypes.c_uint64),
                ("off", u64p), ("nbr", u32p)]


class CCand(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint32), ("pad", ctypes.c_uint32), ("score", ctypes.c_uint64)]


class CParams(ctypes.Structure):
    _fields_ = [("omega", ctypes.c_uint64), ("delta", ctypes.c_uint64), ("pi", ctypes.c_uint32),
                ("norm", ctypes.c_uint32), ("noise_seed", ctypes.c_uint64),
                ("noise_cap", ctypes.c_uint64), ("batch", ctypes.c_uint32)]


CAND_DTYPE = np.dtype([("id", np.uint32), ("pad", np.uint32), ("score", np.uint64)])


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hgp_ref status {code}: {msg}")
        self.code = code
        self.msg = msg


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libhgp_ref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        L = ctypes.CDLL(path)
        L.hgp_ref_build_csr.argtypes = [ctypes.POINTER(CInput), ctypes.POINTER(CCsr)]
        L.hgp_ref_unique_neighbors.argtypes = [ctypes.POINTER(CCsr), ctypes.c_uint32, ctypes.c_uint32,
                                               ctypes.POINTER(CNbrs)]
        L.hgp_ref_score_pairs.argtypes = [ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs),
                                          ctypes.POINTER(CParams), ctypes.c_void_p]
        L.hgp_ref_match.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p,
                                    ctypes.POINTER(ctypes.c_int64)]
        L.hgp_ref_contract.argtypes = [ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs), u32p, u32p,
                                       ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs)]
        for f in (L.hgp_ref_build_csr, L.hgp_ref_unique_neighbors, L.hgp_ref_score_pairs,
                  L.hgp_ref_match, L.hgp_ref_contract):
            f.restype = ctypes.c_int
        L.hgp_ref_csr_free.argtypes = [ctypes.POINTER(CCsr)]
        L.hgp_ref_nbrs_free.argtypes = [ctypes.POINTER(CNbrs)]
        L.hgp_ref_last_error.restype = ctypes.c_char_p
        _LIB = L
    return _LIB


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().hgp_ref_last_error().decode())


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class Csr:
    """Host copy of one level's compressed sparse layout."""

    N: int
    E: int
    edge_off: np.ndarray
    edge_nsrc: np.ndarray
    pins: np.ndarray
    edge_w: np.ndarray
    edge_mu: np.ndarray
    node_w: np.ndarray
    inc_off: np.ndarray
    inc_nin: np.ndarray
    inc: np.ndarray
    in_mu: np.ndarray

    @property
    def P(self) -> int:
        return int(self.pins.shape[0])

    def _c(self) -> CCsr:
        self._keep = [np.ascontiguousarray(a) for a in (
            self.edge_off, self.edge_nsrc, self.pins, self.edge_w, self.edge_mu, self.node_w,
            self.inc_off, self.inc_nin, self.inc, self.in_mu)]
        k = self._keep
        return CCsr(self.N, self.E, self.P, _ptr(k[0], u64p), _ptr(k[1], u32p), _ptr(k[2], u32p),
                    _ptr(k[3], u32p), _ptr(k[4], u32p), _ptr(k[5], u32p), _ptr(k[6], u64p),
                    _ptr(k[7], u32p), _ptr(k[8], u32p), _ptr(k[9], u32p))


@dataclass
class Nbrs:
    lo: int
    hi: int
    off: np.ndarray   # u64 [hi-lo+1]
    nbr: np.ndarray   # u32 [V], bit31 = purge

    def _c(self) -> CNbrs:
        self.off = np.ascontiguousarray(self.off)
        self.nbr = np.ascontiguousarray(self.nbr)
        return CNbrs(self.lo, self.hi, int(self.nbr.shape[0]), _ptr(self.off, u64p), _ptr(self.nbr, u32p))

    def copy(self) -> "Nbrs":
        return Nbrs(self.lo, self.hi, self.off.copy(), self.nbr.copy())

    def segment(self, n: int) -> np.ndarray:
        return self.nbr[int(self.off[n - self.lo]):int(self.off[n - self.lo + 1])]


def _arr(ptr, n, dt):
    if n == 0:
        return np.zeros(0, dtype=dt)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)


def _take_csr(c: CCsr) -> Csr:
    N, E, P = c.N, c.E, c.P
    out = Csr(N, E, _arr(c.edge_off, E + 1, np.uint64), _arr(c.edge_nsrc, E, np.uint32),
              _arr(c.pins, P, np.uint32), _arr(c.edge_w, E, np.uint32), _arr(c.edge_mu, E, np.uint32),
              _arr(c.node_w, N, np.uint32), _arr(c.inc_off, N + 1, np.uint64),
              _arr(c.inc_nin, N, np.uint32), _arr(c.inc, P, np.uint32), _arr(c.in_mu, N, np.uint32))
    lib().hgp_ref_csr_free(ctypes.byref(c))
    return out


def _take_nbrs(c: CNbrs) -> Nbrs:
    out = Nbrs(c.lo, c.hi, _arr(c.off, c.hi - c.lo + 1, np.uint64), _arr(c.nbr, c.V, np.uint32))
    lib().hgp_ref_nbrs_free(ctypes.byref(c))
    return out


def params(omega: int, delta: int, pi: int = 4, norm: int = 0, noise_seed: int = 0,
           noise_cap: int = 0, batch: int = 0) -> CParams:
    return CParams(omega, delta, pi, norm, noise_seed, noise_cap, batch)


def build_csr(num_nodes, edge_off, edge_nsrc, pins, edge_w, node_w) -> Csr:
    arrs = [np.ascontiguousarray(edge_off, dtype=np.uint64), np.ascontiguousarray(edge_nsrc, dtype=np.uint32),
            np.ascontiguousarray(pins, dtype=np.uint32), np.ascontiguousarray(edge_w, dtype=np.uint32),
            np.ascontiguousarray(node_w, dtype=np.uint32)]
    if arrs[0].shape[0] == 0:
        arrs[0] = np.zeros(1, dtype=np.uint64)
    ci = CInput(num_nodes, arrs[1].shape[0], _ptr(arrs[0], u64p), _ptr(arrs[1], u32p), _ptr(arrs[2], u32p),
                _ptr(arrs[3], u32p), _ptr(arrs[4], u32p))
    out = CCsr()
    _check(lib().hgp_ref_build_csr(ctypes.byref(ci), ctypes.byref(out)))
    return _take_csr(out)


def build_csr_hg(hg) -> Csr:
    return build_csr(hg.num_nodes, hg.edge_off, hg.edge_nsrc, hg.pins, hg.edge_w, hg.node_w)


def unique_neighbors(g: Csr, lo: int = 0, hi: int | None = None) -> Nbrs:
    hi = g.N if hi is None else hi
    cg = g._c()
    out = CNbrs()
    _check(lib().hgp_ref_unique_neighbors(ctypes.byref(cg), lo, hi, ctypes.byref(out)))
    return _take_nbrs(out)


def score_pairs(g: Csr, nb: Nbrs, p: CParams) -> np.ndarray:
    """Writes purge flags into ``nb.nbr`` in place; returns cand [N, pi] (rows lo..hi-1 set)."""
    cand = np.zeros((g.N, p.pi), dtype=CAND_DTYPE)
    cand["id"] = NONE
    cg, cn = g._c(), nb._c()
    _check(lib().hgp_ref_score_pairs(ctypes.byref(cg), ctypes.byref(cn), ctypes.byref(p),
                                     cand.ctypes.data_as(ctypes.c_void_p)))
    return cand


def match(cand: np.ndarray, pi: int | None = None):
    """Returns (match [N], matched pairs per round [pi], DP optimum per round [pi])."""
    cand = np.ascontiguousarray(cand, dtype=CAND_DTYPE)
    N = cand.shape[0]
    pi = cand.shape[1] if pi is None else pi
    m = np.zeros(N, dtype=np.uint32)
    per = np.zeros(pi, dtype=np.uint32)
    val = np.zeros(pi, dtype=np.int64)
    _check(lib().hgp_ref_match(cand.ctypes.data_as(ctypes.c_void_p), N, pi, _ptr(m, u32p),
                               _ptr(per, u32p), val.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return m, per, val


def contract(g: Csr, nb: Nbrs, match_arr: np.ndarray):
    """Returns (gamma [N], coarse Csr, coarse Nbrs)."""
    match_arr = np.ascontiguousarray(match_arr, dtype=np.uint32)
    gamma = np.zeros(g.N, dtype=np.uint32)
    cg, cn = g._c(), nb._c()
    oc, on = CCsr(), CNbrs()
    _check(lib().hgp_ref_contract(ctypes.byref(cg), ctypes.byref(cn), _ptr(match_arr, u32p),
                                  _ptr(gamma, u32p), ctypes.byref(oc), ctypes.byref(on)))
    return gamma, _take_csr(oc), _take_nbrs(on)


def coarsen_level(g: Csr, nb: Nbrs, p: CParams, leftover: bool = False):
    """score -> match (-> f2 leftover pairing if asked) -> contract; nb flags are written in place.
    Returns a dict."""
    cand = score_pairs(g, nb, p)
    m, per, val = match(cand, p.pi)
    if leftover:
        m, extra = leftover_pairs(cand, g.node_w, g.in_mu, p.omega, p.delta, m)
    gamma, cg, cnb = contract(g, nb, m)
    return {"cand": cand, "match": m, "matched_per_round": per, "round_value": val,
            "gamma": gamma, "coarse": cg, "coarse_nb": cnb}


def leftover_targets(cand: np.ndarray, node_w: np.ndarray, in_mu: np.ndarray, omega: int, delta: int) -> np.ndarray:
    """SURVEY §8(f) f2, the best-effort pairing of P:673-677 read deterministically (DESIGN
    reading #22). L = the nodes left with no candidate (cand[n][0] = NONE; they have no valid
    neighbour, so a4 never matches them). Each n in L targets, among the other m in L with
    size(n) + size(m) <= Omega and in_mu(n) + in_mu(m) <= Delta (the paper's over-estimate of
    the inbound union), the one with the largest (size(m), m) — "sorted by size ... the
    first valid node it finds", contentions broken by id. Score = size(n) + size(m). Returns a
    [N, 1] candidate array (NONE outside L / without a valid partner). Plain O(|L|^2) loops."""
    N = cand.shape[0]
    out = np.zeros((N, 1), dtype=CAND_DTYPE)
    out["id"] = NONE
    L = [n for n in range(N) if int(cand[n][0]["id"]) == NONE]
    w = [int(x) for x in node_w]
    im = [int(x) for x in in_mu]
    for n in L:
        best = None
        for m in L:
            if m == n or w[n] + w[m] > omega:
                continue
            if delta != UNBOUNDED and im[n] + im[m] > delta:
                continue
            if best is None or (w[m], m) > (w[best], best):
                best = m
        if best is not None:
            out[n, 0] = (best, 0, w[n] + w[best])
    return out


def leftover_pairs(cand: np.ndarray, node_w: np.ndarray, in_mu: np.ndarray, omega: int, delta: int,
                   match_arr: np.ndarray):
    """f2: the targets of leftover_targets solved by the a4 DP as one extra round (pi = 1) and
    merged into match_arr. Returns (match [N], pairs added)."""
    c2 = leftover_targets(cand, node_w, in_mu, omega, delta)
    m2, per2, _ = match(c2, 1)
    out = np.array(match_arr, dtype=np.uint32, copy=True)
    sel = m2 != NONE
    assert np.all(out[sel] == NONE), "a leftover node was already matched"
    out[sel] = m2[sel]
    return out, int(per2[0])


def stop_nodes(g0: Csr, omega: int) -> int:
    """Reading #20 (coarsen until |N| reaches ceil(W/Omega) or no valid cluster is
    left): the node count at or below which the multi-level driver stops; W = total size."""
    W = int(g0.node_w.astype(np.uint64).sum())
    return 1 if omega == UNBOUNDED else max(1, -(-W // int(omega)))


def coarsen(g0: Csr, p: CParams, max_levels: int = 64, leftover: bool = False) -> dict:
    """Multi-level driver, written out plainly: level l is
    coarsen_level on the previous level's coarse CSR and neighbour lists, with noise seed
    p.noise_seed + l (reading #3: "the driver passes seed+level"); it stops after the first level
    whose coarse node count is <= stop_nodes(g0, Omega) or that formed no pair, by a4 or by the f2
    leftover pairing (N' = N; reading #20), or
    after max_levels levels. rho = gamma^L o ... o gamma^1 maps each level-0 node to its node on
    the coarsest level (the initial partition's clusters)."""
    g, nb = g0, unique_neighbors(g0)
    rho = np.arange(g0.N, dtype=np.uint32)
    stop = stop_nodes(g0, p.omega)
    levels = []
    for lvl in range(max_levels):
        pl = params(p.omega, p.delta, p.pi, norm=p.norm, noise_seed=p.noise_seed + lvl, noise_cap=p.noise_cap)
        r = coarsen_level(g, nb, pl, leftover)
        rho = r["gamma"][rho]
        per = [int(x) for x in r["matched_per_round"]]
        cg = r["coarse"]
        levels.append({"N": g.N, "E": g.E, "P": g.P, "Nc": cg.N, "Ec": cg.E, "Pc": cg.P,
                       "matched_per_round": per, "gamma": r["gamma"], "match": r["match"]})
        g, nb = cg, r["coarse_nb"]
        if g.N <= stop or cg.N == levels[-1]["N"]:   # no pair formed (a4 or f2): N' = N
            break
    return {"rho": rho, "levels": levels, "coarsest": g, "coarsest_nb": nb, "stop_nodes": stop}


# ----------------------------------------------------------------------------- next rows (§8(f))
class CQuality(ctypes.Structure):
    _fields_ = [("connectivity", ctypes.c_uint64), ("cut_net", ctypes.c_uint64), ("max_size", ctypes.c_uint64),
                ("max_inbound", ctypes.c_uint64), ("size_violations", ctypes.c_uint32),
                ("inbound_violations", ctypes.c_uint32)]


class CPins(ctypes.Structure):
    _fields_ = [("E", ctypes.c_uint32), ("nnz", ctypes.c_uint64), ("off", u64p), ("part", u32p), ("count", u32p)]


i64p = ctypes.POINTER(ctypes.c_int64)


def _lib2():
    L = lib()
    if not hasattr(L, "_refine_typed"):
        cp = ctypes.POINTER(CCsr)
        L.hgp_ref_partition_metrics.argtypes = [cp, u32p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                                ctypes.POINTER(CQuality)]
        L.hgp_ref_pins_matrix.argtypes = [cp, u32p, ctypes.c_int, ctypes.POINTER(CPins)]
        L.hgp_ref_pins_free.argtypes = [ctypes.POINTER(CPins)]
        L.hgp_ref_propose_moves.argtypes = [cp, u32p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, u32p, i64p]
        L.hgp_ref_in_sequence_gains.argtypes = [cp, u32p, ctypes.c_uint32, u32p, ctypes.c_uint32, u32p, i64p]
        L.hgp_ref_sequence_violations.argtypes = [cp, u32p, ctypes.c_uint32, u32p, ctypes.c_uint32, u32p,
                                                  ctypes.c_uint64, ctypes.c_uint64, u32p]
        L.hgp_ref_best_prefix.argtypes = [i64p, u32p, ctypes.c_uint32, u32p, i64p]
        for f in (L.hgp_ref_partition_metrics, L.hgp_ref_pins_matrix, L.hgp_ref_propose_moves,
                  L.hgp_ref_in_sequence_gains, L.hgp_ref_sequence_violations, L.hgp_ref_best_prefix):
            f.restype = ctypes.c_int
        L._refine_typed = True
    return L


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def partition_metrics(g: Csr, part, nparts: int, omega: int = UNBOUNDED, delta: int = UNBOUNDED) -> dict:
    """f1: Eq.1 connectivity, Eq.16 cut-net and the constraint loads of a partition of g."""
    part = _u32(part)
    q = CQuality()
    cg = g._c()
    _check(_lib2().hgp_ref_partition_metrics(ctypes.byref(cg), _ptr(part, u32p), nparts, omega, delta,
                                             ctypes.byref(q)))
    return {k: int(getattr(q, k)) for k, _ in CQuality._fields_}


def pins_matrix(g: Csr, part, inbound: bool = False):
    """f3: per edge the sorted (partition, count) pairs of pins(p, e) (or pins_in). Returns (off, part, count)."""
    part = _u32(part)
    out = CPins()
    cg = g._c()
    _check(_lib2().hgp_ref_pins_matrix(ctypes.byref(cg), _ptr(part, u32p), int(inbound), ctypes.byref(out)))
    res = (_arr(out.off, out.E + 1, np.uint64), _arr(out.part, out.nnz, np.uint32), _arr(out.count, out.nnz, np.uint32))
    _lib2().hgp_ref_pins_free(ctypes.byref(out))
    return res


def propose_moves(g: Csr, part, nparts: int, omega: int = UNBOUNDED, enforce_size: bool = False):
    """f3: Eq.13 proposals. Returns (dest [N] u32, NONE = no move; gain [N] i64)."""
    part = _u32(part)
    dest = np.zeros(g.N, dtype=np.uint32)
    gain = np.zeros(g.N, dtype=np.int64)
    cg = g._c()
    _check(_lib2().hgp_ref_propose_moves(ctypes.byref(cg), _ptr(part, u32p), nparts, omega, int(enforce_size),
                                         _ptr(dest, u32p), gain.ctypes.data_as(i64p)))
    return dest, gain


def in_sequence_gains(g: Csr, part, nparts: int, seq, dest) -> np.ndarray:
    part, seq, dest = _u32(part), _u32(seq), _u32(dest)
    out = np.zeros(len(seq), dtype=np.int64)
    cg = g._c()
    _check(_lib2().hgp_ref_in_sequence_gains(ctypes.byref(cg), _ptr(part, u32p), nparts, _ptr(seq, u32p), len(seq),
                                             _ptr(dest, u32p), out.ctypes.data_as(i64p)))
    return out


def sequence_violations(g: Csr, part, nparts: int, seq, dest, omega: int, delta: int) -> np.ndarray:
    part, seq, dest = _u32(part), _u32(seq), _u32(dest)
    out = np.zeros(len(seq), dtype=np.uint32)
    cg = g._c()
    _check(_lib2().hgp_ref_sequence_violations(ctypes.byref(cg), _ptr(part, u32p), nparts, _ptr(seq, u32p),
                                               len(seq), _ptr(dest, u32p), omega, delta, _ptr(out, u32p)))
    return out


def best_prefix(gain_seq, violations):
    gs = np.ascontiguousarray(gain_seq, dtype=np.int64)
    vi = _u32(violations)
    k = ctypes.c_uint32()
    b = ctypes.c_int64()
    _check(_lib2().hgp_ref_best_prefix(gs.ctypes.data_as(i64p), _ptr(vi, u32p), len(gs), ctypes.byref(k),
                                       ctypes.byref(b)))
    return int(k.value), int(b.value)
