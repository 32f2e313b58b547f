"""Multi-GPU sharding of the coarsening level and of the multi-level driver (
BASELINE.json north_star: "scoring and matching shard by node range over a replicated CSR,
per-node choices are exchanged with NCCL all-gather, contraction is rebuilt per shard").

One process per GPU. Every rank holds the replicated CSR of the level. Per level:
  a2+a3  sharded by node range [lo, hi) (equal traversal work, hgp_shard_bounds): N(n) and the
         candidate rows of the range only;
  X1     all-gather of the candidate rows (rank order = node order);
  a4     replicated (O(N)): the same match everywhere, then gamma (hgp_gamma);
  a5     coarse edges of the rank's fine EDGE range (hgp_contract_edges, equal pin counts);
  X2     all-gather of the ranges' pre-merge coarse edges (rank order = fine edge id order);
         the parallel-edge merge and the coarse incidence are rebuilt replicated
         (hgp_contract_merge) — the coarse CSR is the next level's replicated CSR;
  X3     halo exchange: coarse node c = {a, b} (a its min member) belongs to the rank owning a;
         when b lives on another rank its N(b) (with a3's purge flags) is sent point-to-point;
  a5'    coarse neighbours of the rank's coarse node range (hgp_coarse_neighbors): the next
         level's sharded N'.
Bit-identical to one GPU by construction: every per-element result depends only on replicated
data, concatenations follow id order, class representatives are global min fine ids.

Collectives go through a Comm: DistComm (torch.distributed: NCCL on GPUs, gloo on CPU) or
LoopbackComm (W logical ranks in one process, one after the other — tests the schedule on one GPU).
This module is plumbing (routing, concatenation, offsets of gathered pieces); every step of the
method runs in libhgp.so kernels.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import hgp

NONE_I32 = -1   # HGP_NONE seen through an int32 view


# ------------------------------------------------------------------------------------ collectives
def allgather_v(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """All-gather 1-D tensors of different lengths (pads to the max length)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    buf = torch.zeros(max(mx, 1), dtype=t.dtype, device=t.device)
    buf[:t.numel()] = t
    outs = [torch.empty(max(mx, 1), dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return [o[:s] for o, s in zip(outs, sizes)]


class LoopbackComm:
    """W logical ranks held by one process: collectives are in-order concatenations."""

    def __init__(self, world: int):
        self.world = world
        self.local = list(range(world))

    def allgather(self, xs: list[torch.Tensor]) -> list[torch.Tensor]:
        return list(xs)

    def alltoall(self, send: list[list[torch.Tensor]]) -> list[list[torch.Tensor]]:
        """send[i][q]: from local rank i to rank q -> recv[i][q]: to local rank i from rank q."""
        return [[send[q][r] for q in range(self.world)] for r in range(self.world)]

    def time(self) -> float:
        torch.cuda.synchronize()
        return time.perf_counter()


class DistComm:
    """One rank per process over torch.distributed (NCCL over NVLink on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local = [self.rank]
        # gloo moves host memory: device tensors are staged through the host (tests, --share-device)
        self.stage = dist.get_backend(group) == "gloo"

    def _out(self, t: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
        return t.to(like.device) if self.stage else t

    def allgather(self, xs: list[torch.Tensor]) -> list[torch.Tensor]:
        x = xs[0].contiguous()
        outs = allgather_v(x.cpu() if self.stage else x, self.group)
        return [self._out(o, x) for o in outs]

    def alltoall(self, send: list[list[torch.Tensor]]) -> list[list[torch.Tensor]]:
        if self.stage:
            dev = send[0][0].device
            recv = DistComm._alltoall(self, [[x.cpu() for x in send[0]]])
            return [[r.to(dev) for r in recv[0]]]
        return DistComm._alltoall(self, send)

    def _alltoall(self, send: list[list[torch.Tensor]]) -> list[list[torch.Tensor]]:
        mine = [x.contiguous() for x in send[0]]
        dev = mine[0].device
        sz = torch.tensor([x.numel() for x in mine], dtype=torch.int64, device=dev)
        allsz = [torch.zeros_like(sz) for _ in range(self.world)]
        dist.all_gather(allsz, sz, group=self.group)
        recv = []
        ops = []
        for q in range(self.world):
            n = int(allsz[q][self.rank].item())
            if q == self.rank:
                recv.append(mine[q])
                continue
            r = torch.empty(n, dtype=mine[0].dtype, device=dev)
            recv.append(r)
            if mine[q].numel():
                ops.append(dist.P2POp(dist.isend, mine[q], q, self.group))
            if n:
                ops.append(dist.P2POp(dist.irecv, r, q, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return [recv]

    def time(self) -> float:
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        return time.perf_counter()


# ------------------------------------------------------------------------------------ host routing
def edge_bounds(edge_off: torch.Tensor, world: int) -> list[int]:
    """[0 = b_0 <= ... <= b_W = E]: contiguous edge ranges of about equal pin counts."""
    off = _i64(edge_off)
    E = off.numel() - 1
    P = int(off[-1].item())
    targets = torch.tensor([(P * r) // world for r in range(1, world)], dtype=torch.int64, device=off.device)
    mid = torch.searchsorted(off, targets).tolist() if world > 1 else []
    b = [0] + [min(int(x), E) for x in mid] + [E]
    for i in range(1, len(b)):
        b[i] = max(b[i], b[i - 1])
    return b


def owner_of(bounds: list[int], ids: torch.Tensor) -> torch.Tensor:
    """Rank owning each node id for contiguous ranges bounds[r] <= id < bounds[r+1]."""
    b = torch.tensor(bounds[1:-1], dtype=torch.int64, device=ids.device)
    return torch.searchsorted(b, ids.to(torch.int64), right=True)


def halo_plan(match_i32: torch.Tensor, bounds: list[int], r: int):
    """Nodes b of rank r's range whose partner a = match[b] < b lives on an earlier rank: their
    N(b) goes to owner(a). Returns (b ids, destination ranks), ascending b."""
    lo, hi = bounds[r], bounds[r + 1]
    m = match_i32[lo:hi].to(torch.int64)
    b = torch.arange(lo, hi, dtype=torch.int64, device=match_i32.device)
    sel = (m != NONE_I32) & (m >= 0) & (m < lo)
    return b[sel], owner_of(bounds, m[sel])


def pack_segments(off: torch.Tensor, nbr: torch.Tensor, lo: int, ids: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Concatenated N(b) segments of the listed nodes (ids >= lo, relative offsets off) and their
    lengths (int64)."""
    off = _i64(off)
    rel = ids - lo
    s = off[rel]
    ln = off[rel + 1] - s
    if ids.numel() == 0:
        return torch.empty(0, dtype=torch.int32, device=nbr.device), ln
    idx = torch.repeat_interleave(s - torch.cumsum(ln, 0) + ln, ln) + torch.arange(int(ln.sum().item()),
                                                                                   device=nbr.device)
    return _i32(nbr)[idx], ln


def halo_message(b: torch.Tensor, ln: torch.Tensor, segs: torch.Tensor) -> torch.Tensor:
    """One int32 message: [k, ids (k), lengths (k), entries]."""
    k = torch.tensor([b.numel()], dtype=torch.int32, device=segs.device)
    return torch.cat([k, b.to(torch.int32), ln.to(torch.int32), segs])


def halo_unpack(msg: torch.Tensor):
    k = int(msg[0].item()) if msg.numel() else 0
    ids = msg[1:1 + k].to(torch.int64)
    ln = msg[1 + k:1 + 2 * k].to(torch.int64)
    return ids, ln, msg[1 + 2 * k:]


def segment_view(N: int, lo: int, hi: int, off: torch.Tensor, nbr: torch.Tensor, halos: list[torch.Tensor]):
    """(seg_start u64 [N], seg_len u32 [N], nbr) for hgp_coarse_neighbors: the range's own segments
    (relative offsets off over nbr) followed by the received halo segments."""
    dev = nbr.device
    start = torch.zeros(N, dtype=torch.int64, device=dev)
    length = torch.zeros(N, dtype=torch.int32, device=dev)
    off = _i64(off)
    start[lo:hi] = off[:-1]
    length[lo:hi] = (off[1:] - off[:-1]).to(torch.int32)
    parts = [_i32(nbr)]
    base = int(off[-1].item()) if off.numel() else 0
    for msg in halos:
        ids, ln, entries = halo_unpack(msg)
        if ids.numel() == 0:
            continue
        st = torch.cumsum(ln, 0) - ln + base
        start[ids] = st
        length[ids] = ln.to(torch.int32)
        parts.append(entries)
        base += int(ln.sum().item())
    return start, length, torch.cat(parts) if len(parts) > 1 else parts[0].contiguous()


def assemble(bounds: list[int], cand_rows: list[torch.Tensor], offs: list[torch.Tensor],
             nbrs: list[torch.Tensor]) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Concatenate per-range results in range order.
    cand_rows[r]: [n_r, pi, 2] u64 (or any [n_r, ...]); offs[r]: [n_r + 1] u64 relative offsets
    (offs[r][0] = 0); nbrs[r]: [V_r] u32. Returns (cand [N, ...], off [N + 1], nbr [V])."""
    cand = torch.cat([_i64(c) for c in cand_rows], dim=0)
    base = 0
    pieces = []
    for r, o in enumerate(offs):
        o = _i64(o)
        pieces.append(o[:-1] + base)
        base += int(o[-1].item())
    dev = offs[0].device
    pieces.append(torch.tensor([base], dtype=torch.int64, device=dev))
    off = torch.cat(pieces)
    nbr = torch.cat([_i32(x) for x in nbrs]) if nbrs else torch.empty(0, dtype=torch.int32, device=dev)
    assert cand.shape[0] == bounds[-1] - bounds[0]
    return cand, off, nbr


class NbrsView:
    """An hgp_nbrs over torch-owned device tensors (not freed by the library)."""

    def __init__(self, off: torch.Tensor, nbr: torch.Tensor, lo: int, hi: int, max_deg: int):
        self.off_t, self.nbr_t = off.contiguous(), nbr.contiguous()
        self.c = hgp.CNbrs(lo, hi, self.nbr_t.numel(), max_deg, 0, ctypes.c_void_p(self.off_t.data_ptr()),
                           ctypes.c_void_p(self.nbr_t.data_ptr()))
        self.V = self.nbr_t.numel()

    def tensors(self) -> dict:
        return {"off": self.off_t, "nbr": self.nbr_t}

    def to_host(self) -> dict:
        return {"off": self.off_t.cpu().numpy().view(np.uint64), "nbr": self.nbr_t.cpu().numpy().view(np.uint32)}

    def free(self):
        pass


def _i32(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int32) if t.dtype == torch.uint32 else t


def _i64(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int64) if t.dtype == torch.uint64 else t


# ------------------------------------------------------------------------------------ the level
@dataclass
class RankState:
    r: int
    lo: int
    hi: int
    nb: object = None          # N(n) of [lo, hi) (hgp.Nbrs), purge flags set by a3


@dataclass
class LevelInfo:
    N: int = 0
    Nc: int = 0
    E: int = 0
    Ec: int = 0
    P: int = 0
    pairs: int = 0
    V: int = 0                               # N(n) entries of this process's ranges (before the level)
    ms: dict = field(default_factory=dict)   # compute / comm split (host wall time around synchronised phases)


def level_sharded(ctx: hgp.Ctx, g: hgp.Csr, p: hgp.CParams, states: list[RankState], comm, first: bool,
                  cand: torch.Tensor, match: torch.Tensor, gamma: torch.Tensor, leftover: bool = False):
    """One coarsening level on W node-range shards (the module docstring's schedule). `states`
    are this process's ranks (one for DistComm, all W for LoopbackComm), each with its node range
    and, unless `first`, its N(n). Returns (coarse CSR (replicated), info); every state's nb
    becomes its coarse range's N' and its [lo, hi) the coarse node range."""
    W, N, pi = comm.world, g.N, p.pi
    info = LevelInfo(N=N, E=g.E, P=g.P)
    t = {"a2a3": 0.0, "X1": 0.0, "a4": 0.0, "a5_edges": 0.0, "X2": 0.0, "a5_merge": 0.0, "X3": 0.0, "a5_nbrs": 0.0}
    t0 = comm.time()
    for s in states:                                                   # a2 + a3 on the range
        if first:
            s.nb = hgp.neighbors_and_scores(ctx, g, p, cand, s.lo, s.hi)
        else:
            hgp.score_pairs(ctx, g, s.nb, p, cand)
    t1 = comm.time()
    t["a2a3"] = t1 - t0
    rows = comm.allgather([_i64(cand[s.lo:s.hi]).reshape(-1).clone() for s in states])   # X1
    _i64(cand).copy_(torch.cat(rows).view(N, pi, 2))
    t2 = comm.time()
    t["X1"] = t2 - t1
    per = torch.zeros(pi, dtype=torch.uint32, device=cand.device)     # a4 (replicated)
    hgp.match(ctx, cand, N, pi, match, per)
    info.pairs = int(per.view(torch.int32).sum().item())
    if leftover:
        info.pairs += hgp.leftover_pairs(ctx, cand, N, pi, g.tensors()["node_w"], g.tensors()["in_mu"], p.omega,
                                         p.delta, match)
    hgp.gamma(ctx, match, N, gamma)
    t3 = comm.time()
    t["a4"] = t3 - t2
    eb = edge_bounds(g.tensors()["edge_off"], W)                     # a5 on the edge ranges
    parts = [hgp.contract_edges(ctx, g, gamma, eb[s.r], eb[s.r + 1]) for s in states]
    t4 = comm.time()
    t["a5_edges"] = t4 - t3
    ga = {k: comm.allgather([_dt(x.tensors()[k]) for x in parts]) for k in ("eid", "fp", "nsrc", "size", "pins")}  # X2
    cat = {k: torch.cat(v) for k, v in ga.items()}       # copies: the parts' library memory is freed next
    del ga
    for x in parts:
        x.free()
    size = cat["size"].to(torch.int64)
    off = torch.zeros(size.numel() + 1, dtype=torch.int64, device=size.device)
    off[1:] = torch.cumsum(size, 0)
    allv = hgp.CedgesView(cat["eid"], cat["fp"], cat["nsrc"], cat["size"], off, cat["pins"])
    t5 = comm.time()
    t["X2"] = t5 - t4
    coarse = hgp.contract_merge(ctx, g, match, gamma, allv)          # replicated merge + incidence
    del allv
    t6 = comm.time()
    t["a5_merge"] = t6 - t5
    nbounds = [0] * (W + 1)
    for s in states:
        nbounds[s.r], nbounds[s.r + 1] = s.lo, s.hi
    if len(states) == 1 and W > 1:   # every rank's bounds are needed: all-gather the range starts
        lo_all = comm.allgather([torch.tensor([states[0].lo, states[0].hi], dtype=torch.int64, device=cand.device)])
        nbounds = [int(x[0].item()) for x in lo_all] + [int(lo_all[-1][1].item())]
    cb = hgp.coarse_bounds(ctx, match, N, nbounds)
    m32 = _i32(match)
    send = []
    for s in states:                                                  # X3: the halo exchange
        nb = s.nb.tensors()
        b, dst = halo_plan(m32, nbounds, s.r)
        msgs = []
        for q in range(W):
            sel = b[dst == q]
            segs, ln = pack_segments(nb["off"], nb["nbr"], s.lo, sel)
            msgs.append(halo_message(sel, ln, segs))
        send.append(msgs)
    recv = comm.alltoall(send)
    t7 = comm.time()
    t["X3"] = t7 - t6
    for i, s in enumerate(states):                                    # a5' coarse neighbours
        nb = s.nb.tensors()
        start, length, nbr_all = segment_view(N, s.lo, s.hi, nb["off"], nb["nbr"], recv[i])
        cnb = hgp.coarse_neighbors(ctx, match, gamma, N, start, length, nbr_all, cb[s.r], cb[s.r + 1])
        info.V += int(s.nb.V)
        s.nb.free()
        s.nb, s.lo, s.hi = cnb, cb[s.r], cb[s.r + 1]
    t8 = comm.time()
    t["a5_nbrs"] = t8 - t7
    info.Nc, info.Ec = coarse.N, coarse.E
    info.ms = {k: round(v * 1e3, 3) for k, v in t.items()}
    return coarse, info


def _dt(t: torch.Tensor) -> torch.Tensor:
    """Collective-friendly dtype views (NCCL / gloo have no unsigned 32/64-bit types)."""
    return _i32(_i64(t)).contiguous()


def coarsen_sharded(ctx: hgp.Ctx, g0: hgp.Csr, p: hgp.CParams, comm, max_levels: int = hgp.MAX_LEVELS):
    """The multi-level driver (f1) on W node-range shards: the same levels, stop rule (reading #21),
    noise seeds (seed + level, reading #3) and f2 flag as hgp_coarsen. Returns (rho [N0] (the
    level-0 node -> coarsest node map), levels: list of LevelInfo, coarsest CSR
    (replicated), states holding the coarsest level's sharded N')."""
    W = comm.world
    leftover = bool(p.flags & hgp.FLAG_LEFTOVER)
    bounds = hgp.shard_bounds(ctx, g0, W)
    states = [RankState(r, bounds[r], bounds[r + 1]) for r in comm.local]
    W_total = int(g0.tensors()["node_w"].to(torch.int64).sum().item())
    stop_n = 1 if p.omega >= hgp.UNBOUNDED else -(-W_total // p.omega)
    g, levels = g0, []
    seed = p.noise_seed
    rho = torch.arange(g0.N, dtype=torch.int64, device="cuda")
    for lv in range(max_levels):
        N = g.N
        pl = hgp.params(p.omega, p.delta, p.pi, p.norm, seed + lv, p.noise_cap, p.batch, p.flags)
        cand = hgp.empty_cand(N, p.pi)
        match = torch.empty(N, dtype=torch.uint32, device="cuda")
        gam = torch.empty(N, dtype=torch.uint32, device="cuda")
        coarse, info = level_sharded(ctx, g, pl, states, comm, lv == 0, cand, match, gam, leftover=leftover)
        levels.append(info)
        rho = _i32(gam).to(torch.int64)[rho]                          # rho = gamma o rho
        if g is not g0:
            g.free()
        g = coarse
        if coarse.N <= stop_n or info.pairs == 0:
            break
    return rho.to(torch.int32).view(torch.uint32), levels, g, states
