"""Multi-GPU sharding of one coarsening level (BASELINE.json north_star: "scoring and matching
shard by node range over a replicated CSR, per-node choices are exchanged with NCCL all-gather").

One process per GPU. Every rank holds the replicated level-0 CSR (a1). The node range [0, N) is
split into equal-work contiguous ranges (hgp_shard_bounds, a function of the replicated CSR only,
so every rank computes the same split). Rank r runs the fused a2+a3 on its range; the candidate
rows and the neighbour segments are all-gathered (torch.distributed; NCCL over NVLink on GPUs,
gloo in the CPU tests); a4 and a5 then run identically on every rank. Results are bit-identical
to the single-GPU level: every per-node output depends only on the replicated CSR, and the
all-gather concatenates in rank order = node order.

This module is plumbing (argument marshalling and collectives); every step of the method runs
in libhgp.so kernels.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import hgp


def allgather_v(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """All-gather 1-D tensors of different lengths (pads to the max length)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    buf = torch.zeros(mx, dtype=t.dtype, device=t.device)
    buf[:t.numel()] = t
    outs = [torch.empty(mx, dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return [o[:s] for o, s in zip(outs, sizes)]


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

    def to_host(self) -> dict:
        return {"off": self.off_t.cpu().numpy().view(np.uint64), "nbr": self.nbr_t.cpu().numpy().view(np.uint32)}

    def free(self):
        pass


def _i32(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int32) if t.dtype == torch.uint32 else t


def _i64(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int64) if t.dtype == torch.uint64 else t


def level0_sharded(ctx: hgp.Ctx, g: hgp.Csr, p: hgp.CParams, cand: torch.Tensor, match: torch.Tensor,
                   gamma: torch.Tensor, group=None):
    """The first level on W GPUs: sharded fused a2+a3, all-gathers, replicated a4 + a5.
    Returns (nb_full, coarse, coarse_nb, info)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = hgp.shard_bounds(ctx, g, world)
    lo, hi = bounds[rank], bounds[rank + 1]
    nb_local = hgp.neighbors_and_scores(ctx, g, p, cand, lo, hi)
    loc = nb_local.tensors()
    # candidate rows (u64 pairs) and neighbour segments, in rank order
    rows = _i64(cand[lo:hi]).reshape(-1).contiguous()
    all_rows = allgather_v(rows, group)
    all_off = allgather_v(_i64(loc["off"]).contiguous(), group)
    all_nbr = allgather_v(_i32(loc["nbr"]).contiguous(), group)
    md = torch.tensor([nb_local.c.max_deg], dtype=torch.int64, device=cand.device)
    dist.all_reduce(md, op=dist.ReduceOp.MAX, group=group)
    pi = cand.shape[1]
    cand_full, off, nbr = assemble(bounds, [r.view(-1, pi, 2) for r in all_rows], all_off, all_nbr)
    _i64(cand).copy_(cand_full)
    nb_local.free()
    nb_full = NbrsView(off, nbr, 0, g.N, int(md.item()))
    per = torch.zeros(pi, dtype=torch.uint32, device=cand.device)
    hgp.match(ctx, cand, g.N, pi, match, per)
    coarse, coarse_nb = hgp.contract(ctx, g, nb_full, match, gamma)
    return nb_full, coarse, coarse_nb, {"bounds": bounds, "range": (lo, hi)}


def level0_loopback(ctx: hgp.Ctx, g: hgp.Csr, p: hgp.CParams, cand: torch.Tensor, match: torch.Tensor,
                    gamma: torch.Tensor, world: int):
    """The same sharded schedule with W logical ranks run one after the other on one GPU and the
    all-gathers replaced by the same in-order concatenation (assemble) — tests the sharding
    logic without W GPUs."""
    bounds = hgp.shard_bounds(ctx, g, world)
    rows, offs, nbrs, mds = [], [], [], []
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        nb_r = hgp.neighbors_and_scores(ctx, g, p, cand, lo, hi)
        t = nb_r.tensors()
        rows.append(cand[lo:hi].clone())
        offs.append(t["off"].clone())
        nbrs.append(t["nbr"].clone())
        mds.append(nb_r.c.max_deg)
        nb_r.free()
    cand_full, off, nbr = assemble(bounds, rows, offs, nbrs)
    _i64(cand).copy_(cand_full)
    nb_full = NbrsView(off, nbr, 0, g.N, max(mds))
    pi = cand.shape[1]
    hgp.match(ctx, cand, g.N, pi, match, None)
    coarse, coarse_nb = hgp.contract(ctx, g, nb_full, match, gamma)
    return nb_full, coarse, coarse_nb, bounds
