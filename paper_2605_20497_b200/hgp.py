"""Thin ctypes binding of the C-ABI in include/hgp.h (libhgp.so, sm_100a).

Argument marshalling only: every step of the level runs in the CUDA kernels of
libhgp.so. PyTorch supplies device memory (the library's allocator callback is
``torch.cuda.caching_allocator_alloc``), the stream and the process group.
There is no CPU fallback: without the built extension or a CUDA device every
call raises.
"""
from __future__ import annotations

import contextlib
import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhgp.so")

NONE = 0xFFFFFFFF
UNBOUNDED = (1 << 64) - 1
PURGE = 0x80000000
FP_SHIFT = 24
MAX_PI = 16

u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
vp = ctypes.c_void_p

STATUS = {0: "HGP_OK", -1: "HGP_E_ARG", -2: "HGP_E_MALFORMED", -3: "HGP_E_INFEASIBLE", -4: "HGP_E_OVERFLOW",
          -5: "HGP_E_OOM", -6: "HGP_E_CUDA", -7: "HGP_E_NCCL", -8: "HGP_E_INTERNAL"}


class HgpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class CInput(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_uint32), ("num_edges", ctypes.c_uint32), ("edge_off", vp),
                ("edge_nsrc", vp), ("pins", vp), ("edge_w", vp), ("node_w", vp)]


class CCsr(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint32), ("E", ctypes.c_uint32), ("P", ctypes.c_uint64),
                ("max_edge", ctypes.c_uint32), ("max_inc", ctypes.c_uint32),
                ("edge_off", vp), ("edge_nsrc", vp), ("pins", vp), ("edge_w", vp), ("edge_mu", vp),
                ("node_w", vp), ("inc_off", vp), ("inc_nin", vp), ("inc", vp), ("in_mu", vp)]


class CNbrs(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_uint32), ("hi", ctypes.c_uint32), ("V", ctypes.c_uint64),
                ("max_deg", ctypes.c_uint32), ("pad_", ctypes.c_uint32), ("off", vp), ("nbr", vp)]


class CParams(ctypes.Structure):
    _fields_ = [("omega", ctypes.c_uint64), ("delta", ctypes.c_uint64), ("pi", ctypes.c_uint32),
                ("norm", ctypes.c_uint32), ("noise_seed", ctypes.c_uint64), ("noise_cap", ctypes.c_uint64),
                ("batch", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


class CStats(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint32), ("E", ctypes.c_uint32), ("Nc", ctypes.c_uint32), ("Ec", ctypes.c_uint32),
                ("P", ctypes.c_uint64), ("V", ctypes.c_uint64), ("Pc", ctypes.c_uint64), ("Vc", ctypes.c_uint64),
                ("matched_per_round", ctypes.c_uint32 * MAX_PI), ("dropped_edges", ctypes.c_uint32),
                ("merged_edges", ctypes.c_uint32), ("purged", ctypes.c_uint64), ("ms", ctypes.c_float * 4)]

    def as_dict(self, pi: int = MAX_PI) -> dict:
        return {"N": self.N, "E": self.E, "Nc": self.Nc, "Ec": self.Ec, "P": self.P, "V": self.V, "Pc": self.Pc,
                "Vc": self.Vc, "matched_per_round": list(self.matched_per_round)[:pi],
                "dropped_edges": self.dropped_edges, "merged_edges": self.merged_edges, "purged": self.purged,
                "ms": {"score": self.ms[0], "match": self.ms[1], "contract": self.ms[2], "total": self.ms[3]}}


class CQuality(ctypes.Structure):
    _fields_ = [("connectivity", ctypes.c_uint64), ("cut_net", ctypes.c_uint64), ("max_size", ctypes.c_uint64),
                ("max_inbound", ctypes.c_uint64), ("size_violations", ctypes.c_uint32),
                ("inbound_violations", ctypes.c_uint32)]


class CPins(ctypes.Structure):
    _fields_ = [("E", ctypes.c_uint32), ("pad_", ctypes.c_uint32), ("nnz", ctypes.c_uint64), ("off", vp),
                ("part", vp), ("count", vp)]


class CCedges(ctypes.Structure):
    _fields_ = [("K", ctypes.c_uint32), ("pad_", ctypes.c_uint32), ("P", ctypes.c_uint64), ("eid", vp), ("fp", vp),
                ("nsrc", vp), ("size", vp), ("off", vp), ("pins", vp)]


ALLOC_FN = ctypes.CFUNCTYPE(vp, vp, ctypes.c_size_t, vp)
FREE_FN = ctypes.CFUNCTYPE(None, vp, vp, ctypes.c_size_t, vp)


class CAllocator(ctypes.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", vp)]


CAND_DTYPE = np.dtype([("id", np.uint32), ("pad", np.uint32), ("score", np.uint64)])

_LIB = None


def lib():
    """Load libhgp.so; raises if the CUDA extension was not built (no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() or `make cuda`")
        L = ctypes.CDLL(LIB_PATH)
        S = ctypes.c_int
        L.hgp_ctx_create.argtypes = [ctypes.c_int, vp, ctypes.POINTER(CAllocator), ctypes.POINTER(vp)]
        L.hgp_ctx_destroy.argtypes = [vp]
        L.hgp_last_error.restype = ctypes.c_char_p
        L.hgp_launch_count.argtypes = [vp]
        L.hgp_launch_count.restype = ctypes.c_uint64
        L.hgp_copy.argtypes = [vp, vp, vp, ctypes.c_size_t]
        L.hgp_sync.argtypes = [vp]
        L.hgp_ctx_set_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        L.hgp_ctx_set_option.restype = S
        L.hgp_profile_begin.argtypes = [vp, ctypes.c_char_p]
        L.hgp_profile_end.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
        L.hgp_profile_begin.restype = S
        L.hgp_profile_report.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
        L.hgp_profile_report.restype = S
        L.hgp_profile_end.restype = S
        L.hgp_build_csr.argtypes = [vp, ctypes.POINTER(CInput), ctypes.POINTER(CCsr)]
        L.hgp_unique_neighbors.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.POINTER(CNbrs)]
        L.hgp_score_pairs.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs), ctypes.POINTER(CParams), vp]
        L.hgp_match.argtypes = [vp, vp, ctypes.c_uint32, ctypes.c_uint32, vp, vp]
        L.hgp_contract.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs), vp, vp, ctypes.POINTER(CCsr),
                                   ctypes.POINTER(CNbrs)]
        L.hgp_coarsen_level.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs), ctypes.POINTER(CParams), vp,
                                        vp, vp, ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs), ctypes.POINTER(CStats)]
        L.hgp_coarsen.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.POINTER(CParams), ctypes.c_uint32, vp,
                                  ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs), vp, ctypes.POINTER(ctypes.c_uint32)]
        L.hgp_coarsen.restype = S
        L.hgp_leftover_pairs.argtypes = [vp, vp, ctypes.c_uint32, ctypes.c_uint32, vp, vp, ctypes.c_uint64,
                                         ctypes.c_uint64, vp, vp]
        L.hgp_leftover_pairs.restype = S
        L.hgp_neighbors_and_scores.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.POINTER(CParams), ctypes.c_uint32,
                                               ctypes.c_uint32, ctypes.POINTER(CNbrs), vp]
        L.hgp_shard_bounds.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
        L.hgp_shard_bounds.restype = S
        L.hgp_coarsen_level0.argtypes = [vp, ctypes.POINTER(CCsr), ctypes.POINTER(CParams), vp, vp, vp,
                                         ctypes.POINTER(CNbrs), ctypes.POINTER(CCsr), ctypes.POINTER(CNbrs),
                                         ctypes.POINTER(CStats)]
        L.hgp_csr_free.argtypes = [vp, ctypes.POINTER(CCsr)]
        L.hgp_nbrs_free.argtypes = [vp, ctypes.POINTER(CNbrs)]
        cp, pp = ctypes.POINTER(CCsr), ctypes.POINTER(CPins)
        L.hgp_pins_matrix.argtypes = [vp, cp, vp, ctypes.c_uint32, ctypes.c_int, pp]
        L.hgp_pins_free.argtypes = [vp, pp]
        L.hgp_partition_metrics.argtypes = [vp, cp, vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.POINTER(CQuality), vp, vp]
        L.hgp_propose_moves.argtypes = [vp, cp, vp, ctypes.c_uint32, pp, ctypes.c_uint64, ctypes.c_int, vp, vp]
        L.hgp_in_sequence_gains.argtypes = [vp, cp, vp, ctypes.c_uint32, pp, vp, ctypes.c_uint32, vp, vp]
        L.hgp_sequence_violations.argtypes = [vp, cp, vp, ctypes.c_uint32, pp, vp, ctypes.c_uint32, vp,
                                              ctypes.c_uint64, ctypes.c_uint64, vp]
        L.hgp_best_prefix.argtypes = [vp, vp, vp, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
                                      ctypes.POINTER(ctypes.c_int64)]
        L.hgp_gamma.argtypes = [vp, vp, ctypes.c_uint32, vp, ctypes.POINTER(ctypes.c_uint32)]
        L.hgp_coarse_bounds.argtypes = [vp, vp, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32,
                                        ctypes.POINTER(ctypes.c_uint32)]
        L.hgp_contract_edges.argtypes = [vp, ctypes.POINTER(CCsr), vp, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.POINTER(CCedges)]
        L.hgp_cedges_free.argtypes = [vp, ctypes.POINTER(CCedges)]
        L.hgp_contract_merge.argtypes = [vp, ctypes.POINTER(CCsr), vp, vp, ctypes.POINTER(CCedges), ctypes.POINTER(CCsr)]
        L.hgp_coarse_neighbors.argtypes = [vp, vp, vp, ctypes.c_uint32, vp, vp, vp, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.POINTER(CNbrs)]
        for f in (L.hgp_gamma, L.hgp_coarse_bounds, L.hgp_contract_edges, L.hgp_contract_merge, L.hgp_coarse_neighbors):
            f.restype = S
        L.hgp_tier_counts.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        L.hgp_tier_counts.restype = S
        for f in (L.hgp_pins_matrix, L.hgp_partition_metrics, L.hgp_propose_moves, L.hgp_in_sequence_gains,
                  L.hgp_sequence_violations, L.hgp_best_prefix):
            f.restype = S
        for f in (L.hgp_ctx_create, L.hgp_copy, L.hgp_sync, L.hgp_build_csr, L.hgp_unique_neighbors,
                  L.hgp_score_pairs, L.hgp_match, L.hgp_contract, L.hgp_coarsen_level,
                  L.hgp_neighbors_and_scores, L.hgp_coarsen_level0):
            f.restype = S
        _LIB = L
    return _LIB


def exported_symbols() -> list[str]:
    """Names of every hgp_* function declared in include/hgp.h (used by the CPU-side ABI test)."""
    import re
    hdr = open(os.path.join(os.path.dirname(_HERE), "include", "hgp.h")).read()
    return sorted(set(re.findall(r"HGP_API\s+[\w\s\*]+?\b(hgp_\w+)\s*\(", hdr)))


def _check(rc: int):
    if rc != 0:
        raise HgpError(rc, lib().hgp_last_error().decode())


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory (zero copy)."""

    def __init__(self, ptr: int, n: int, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None}
        self._owner = owner


def dev_view(ptr, n: int, dtype: str, owner=None) -> torch.Tensor:
    typestr = {"u32": "<u4", "u64": "<u8", "u8": "|u1"}[dtype]
    if n == 0 or not ptr:
        tdt = {"u32": torch.uint32, "u64": torch.uint64, "u8": torch.uint8}[dtype]
        return torch.empty(0, dtype=tdt, device="cuda")
    return torch.as_tensor(_DevArray(int(ptr), int(n), typestr, owner), device="cuda")


class Ctx:
    """One library context: device, stream, allocator (torch caching allocator by default)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None, allocator: str = "torch"):
        if not torch.cuda.is_available():
            raise RuntimeError("hgp: no CUDA device; the product path has no CPU fallback")
        self.device = device
        self.stream = stream or torch.cuda.current_stream(device)
        self._alloc = None
        if allocator == "torch":
            dev, st = device, self.stream

            def _a(user, nbytes, stream):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st)
                except Exception:   # OOM -> NULL -> HGP_E_OOM
                    return None

            def _f(user, ptr, nbytes, stream):
                if ptr:
                    torch.cuda.caching_allocator_delete(int(ptr))

            self._afn, self._ffn = ALLOC_FN(_a), FREE_FN(_f)
            self._alloc = CAllocator(self._afn, self._ffn, None)
        h = vp()
        _check(lib().hgp_ctx_create(device, vp(self.stream.cuda_stream),
                                    ctypes.byref(self._alloc) if self._alloc else None, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().hgp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().hgp_launch_count(self.h))

    def sync(self):
        _check(lib().hgp_sync(self.h))

    OPTION_DEFAULTS = {"fused_sample_min": 65536, "fused_pool_cap": 0, "unfused": 0, "inc_radix": 0,
                       "debug_sync": 0, "no_hub": 0}

    def set_option(self, name: str, value: int):
        """hgp_ctx_set_option (tests / experiments; results never depend on options)."""
        _check(lib().hgp_ctx_set_option(self.h, name.encode(), int(value)))

    @contextlib.contextmanager
    def options(self, **kw):
        """Set options for a with-block and restore their defaults afterwards."""
        for k, v in kw.items():
            self.set_option(k, v)
        try:
            yield self
        finally:
            for k in kw:
                self.set_option(k, self.OPTION_DEFAULTS[k])

    def profile_begin(self, name_filter: str):
        _check(lib().hgp_profile_begin(self.h, name_filter.encode()))

    def profile_end(self):
        """(summed device ms, launches) of the kernels matched since profile_begin."""
        ms, n = ctypes.c_double(), ctypes.c_uint64()
        _check(lib().hgp_profile_end(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def profile_report(self) -> dict:
        """{kernel name: (ms, launches)} for the launches recorded by the last profile window."""
        buf = ctypes.create_string_buffer(1 << 16)
        _check(lib().hgp_profile_report(self.h, buf, len(buf)))
        out = {}
        for item in buf.value.decode().split(";"):
            if item:
                name, ms, n = item.rsplit(":", 2)
                out[name] = (float(ms), int(n))
        return out

    TIERS = ["fused_S", "fused_A", "fused_M", "fused_B", "nbrs_1", "nbrs_2", "nbrs_3", "score_nointer",
             "score_packed", "score_split", "score_B", "score_W", "score_H", "cnbrs_A", "cnbrs_M", "cnbrs_B",
             "cnbrs_C", "jump", "fused_W", "fused_H", "cnbrs_H", "cnbrs_A2", "score_hub"]

    def tier_counts(self, reset: bool = False) -> dict:
        """hgp_tier_counts: nodes processed per kernel tier (include/hgp.h HGP_TIER_*)."""
        arr = (ctypes.c_uint64 * 24)()
        _check(lib().hgp_tier_counts(self.h, arr, int(reset)))
        return {name: int(arr[i]) for i, name in enumerate(self.TIERS)}

    def copy(self, dst_ptr: int, src_ptr: int, nbytes: int):
        _check(lib().hgp_copy(self.h, vp(dst_ptr), vp(src_ptr), nbytes))


FLAG_LEFTOVER = 1   # hgp_params.flags: f2 leftover pairing after a4


def params(omega: int, delta: int, pi: int = 4, norm: int = 0, noise_seed: int = 0, noise_cap: int = 0,
           batch: int = 0, flags: int = 0) -> CParams:
    return CParams(omega, delta, pi, norm, noise_seed, noise_cap, batch, flags)


class Csr:
    """A level owned by the library (freed with hgp_csr_free)."""

    def __init__(self, ctx: Ctx, c: CCsr):
        self.ctx, self.c = ctx, c

    N = property(lambda s: s.c.N)
    E = property(lambda s: s.c.E)
    P = property(lambda s: s.c.P)

    def tensors(self) -> dict:
        c = self.c
        N, E, P = c.N, c.E, c.P
        return {"edge_off": dev_view(c.edge_off, E + 1, "u64", self), "edge_nsrc": dev_view(c.edge_nsrc, E, "u32", self),
                "pins": dev_view(c.pins, P, "u32", self), "edge_w": dev_view(c.edge_w, E, "u32", self),
                "edge_mu": dev_view(c.edge_mu, E, "u32", self), "node_w": dev_view(c.node_w, N, "u32", self),
                "inc_off": dev_view(c.inc_off, N + 1, "u64", self), "inc_nin": dev_view(c.inc_nin, N, "u32", self),
                "inc": dev_view(c.inc, P, "u32", self), "in_mu": dev_view(c.in_mu, N, "u32", self)}

    def to_host(self) -> dict:
        return {k: v.cpu().numpy() for k, v in self.tensors().items()}

    def free(self):
        if self.c is not None and self.ctx.h:
            lib().hgp_csr_free(self.ctx.h, ctypes.byref(self.c))
        self.c = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Nbrs:
    def __init__(self, ctx: Ctx, c: CNbrs):
        self.ctx, self.c = ctx, c

    lo = property(lambda s: s.c.lo)
    hi = property(lambda s: s.c.hi)
    V = property(lambda s: s.c.V)

    def tensors(self) -> dict:
        c = self.c
        return {"off": dev_view(c.off, c.hi - c.lo + 1, "u64", self), "nbr": dev_view(c.nbr, c.V, "u32", self)}

    def to_host(self) -> dict:
        return {k: v.cpu().numpy() for k, v in self.tensors().items()}

    def free(self):
        if self.c is not None and self.ctx.h:
            lib().hgp_nbrs_free(self.ctx.h, ctypes.byref(self.c))
        self.c = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _ptr(t: torch.Tensor | None) -> vp:
    return vp(t.data_ptr()) if t is not None else vp()


def input_struct(num_nodes: int, edge_off: torch.Tensor, edge_nsrc: torch.Tensor, pins: torch.Tensor,
                 edge_w: torch.Tensor, node_w: torch.Tensor) -> CInput:
    return CInput(num_nodes, edge_nsrc.numel(), _ptr(edge_off), _ptr(edge_nsrc), _ptr(pins), _ptr(edge_w),
                  _ptr(node_w))


def build_csr(ctx: Ctx, num_nodes: int, edge_off, edge_nsrc, pins, edge_w, node_w) -> Csr:
    """a1 on DEVICE tensors (u64/u32 torch tensors on ctx's device)."""
    ci = input_struct(num_nodes, edge_off, edge_nsrc, pins, edge_w, node_w)
    out = CCsr()
    _check(lib().hgp_build_csr(ctx.h, ctypes.byref(ci), ctypes.byref(out)))
    return Csr(ctx, out)


def unique_neighbors(ctx: Ctx, g: Csr, lo: int = 0, hi: int | None = None) -> Nbrs:
    hi = g.N if hi is None else hi
    out = CNbrs()
    _check(lib().hgp_unique_neighbors(ctx.h, ctypes.byref(g.c), lo, hi, ctypes.byref(out)))
    return Nbrs(ctx, out)


def empty_cand(N: int, pi: int, device="cuda") -> torch.Tensor:
    """[N, pi] hgp_cand array as a u64 tensor of shape [N, pi, 2] (id|pad, score)."""
    return torch.empty((N, pi, 2), dtype=torch.uint64, device=device)


def score_pairs(ctx: Ctx, g: Csr, nb: Nbrs, p: CParams, cand: torch.Tensor):
    _check(lib().hgp_score_pairs(ctx.h, ctypes.byref(g.c), ctypes.byref(nb.c), ctypes.byref(p), _ptr(cand)))


def match(ctx: Ctx, cand: torch.Tensor, N: int, pi: int, out: torch.Tensor, per_round: torch.Tensor | None = None):
    _check(lib().hgp_match(ctx.h, _ptr(cand), N, pi, _ptr(out), _ptr(per_round)))


def contract(ctx: Ctx, g: Csr, nb: Nbrs, match_t: torch.Tensor, gamma: torch.Tensor):
    oc, on = CCsr(), CNbrs()
    _check(lib().hgp_contract(ctx.h, ctypes.byref(g.c), ctypes.byref(nb.c), _ptr(match_t), _ptr(gamma),
                              ctypes.byref(oc), ctypes.byref(on)))
    return Csr(ctx, oc), Nbrs(ctx, on)


def coarsen_level(ctx: Ctx, g: Csr, nb: Nbrs, p: CParams, cand: torch.Tensor | None, match_t: torch.Tensor,
                  gamma: torch.Tensor):
    oc, on, st = CCsr(), CNbrs(), CStats()
    _check(lib().hgp_coarsen_level(ctx.h, ctypes.byref(g.c), ctypes.byref(nb.c), ctypes.byref(p), _ptr(cand),
                                   _ptr(match_t), _ptr(gamma), ctypes.byref(oc), ctypes.byref(on), ctypes.byref(st)))
    return Csr(ctx, oc), Nbrs(ctx, on), st.as_dict(p.pi)


def neighbors_and_scores(ctx: Ctx, g: Csr, p: CParams, cand: torch.Tensor, lo: int = 0, hi: int | None = None) -> Nbrs:
    """Fused a2 + a3 on nodes [lo, hi) of a level without flags (level 0)."""
    hi = g.N if hi is None else hi
    out = CNbrs()
    _check(lib().hgp_neighbors_and_scores(ctx.h, ctypes.byref(g.c), ctypes.byref(p), lo, hi, ctypes.byref(out),
                                          _ptr(cand)))
    return Nbrs(ctx, out)


def shard_bounds(ctx: Ctx, g: Csr, world: int) -> list[int]:
    """[0 = b_0 <= b_1 <= ... <= b_world = N]: equal-work contiguous node ranges."""
    arr = (ctypes.c_uint32 * (world + 1))()
    _check(lib().hgp_shard_bounds(ctx.h, ctypes.byref(g.c), world, arr))
    return list(arr)


def coarsen_level0(ctx: Ctx, g: Csr, p: CParams, cand: torch.Tensor | None, match_t: torch.Tensor,
                   gamma: torch.Tensor, want_nbrs: bool = True):
    """First level from a level-0 CSR: fused a2+a3, a4, a5. Returns (nb, coarse, coarse_nb, stats);
    nb is None when want_nbrs is False (N(n) is then consumed in place by a5)."""
    nb, oc, on, st = CNbrs(), CCsr(), CNbrs(), CStats()
    _check(lib().hgp_coarsen_level0(ctx.h, ctypes.byref(g.c), ctypes.byref(p), _ptr(cand), _ptr(match_t),
                                    _ptr(gamma), ctypes.byref(nb) if want_nbrs else None, ctypes.byref(oc),
                                    ctypes.byref(on), ctypes.byref(st)))
    return (Nbrs(ctx, nb) if want_nbrs else None), Csr(ctx, oc), Nbrs(ctx, on), st.as_dict(p.pi)


MAX_LEVELS = 64


def leftover_pairs(ctx: Ctx, cand: torch.Tensor, N: int, pi: int, node_w: torch.Tensor, in_mu: torch.Tensor,
                   omega: int, delta: int, match_t: torch.Tensor) -> int:
    """f2 (hgp_leftover_pairs): pairs the nodes left without candidates; extends match_t in place.
    Returns the number of pairs added."""
    added = torch.zeros(1, dtype=torch.uint32, device="cuda")
    _check(lib().hgp_leftover_pairs(ctx.h, _ptr(cand), N, pi, _ptr(node_w), _ptr(in_mu), omega, delta,
                                    _ptr(match_t), _ptr(added)))
    return int(added.item())


def coarsen(ctx: Ctx, g: Csr, p: CParams, max_levels: int = MAX_LEVELS):
    """Multi-level driver (hgp_coarsen): returns (rho [N0] u32 device tensor,
    coarsest Csr, coarsest Nbrs, per-level stats dicts)."""
    rho = torch.empty(g.N, dtype=torch.uint32, device="cuda")
    oc, on = CCsr(), CNbrs()
    st = (CStats * max_levels)()
    nl = ctypes.c_uint32(0)
    _check(lib().hgp_coarsen(ctx.h, ctypes.byref(g.c), ctypes.byref(p), max_levels, _ptr(rho), ctypes.byref(oc),
                             ctypes.byref(on), ctypes.cast(st, vp), ctypes.byref(nl)))
    return rho, Csr(ctx, oc), Nbrs(ctx, on), [st[i].as_dict(p.pi) for i in range(nl.value)]


def cand_to_numpy(cand: torch.Tensor) -> np.ndarray:
    """[N, pi, 2] u64 device tensor -> structured numpy array with fields (id, pad, score)."""
    raw = cand.cpu().numpy().reshape(cand.shape[0], cand.shape[1], 2)
    out = np.zeros(raw.shape[:2], dtype=CAND_DTYPE)
    out["id"] = (raw[..., 0] & 0xFFFFFFFF).astype(np.uint32)
    out["pad"] = (raw[..., 0] >> 32).astype(np.uint32)
    out["score"] = raw[..., 1]
    return out


# ---- rows after the level: f1 quality, f3 refinement gains, f4 validation --------

class Pins:
    """A pins(p, e) / pins_in(p, e) matrix owned by the library (hgp_pins_free)."""

    def __init__(self, ctx: Ctx, c: CPins):
        self.ctx, self.c = ctx, c

    nnz = property(lambda s: s.c.nnz)

    def tensors(self) -> dict:
        c = self.c
        return {"off": dev_view(c.off, c.E + 1, "u64", self), "part": dev_view(c.part, c.nnz, "u32", self),
                "count": dev_view(c.count, c.nnz, "u32", self)}

    def to_host(self) -> dict:
        return {k: v.cpu().numpy() for k, v in self.tensors().items()}

    def free(self):
        if self.c is not None and self.ctx.h:
            lib().hgp_pins_free(self.ctx.h, ctypes.byref(self.c))
        self.c = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _pins_ref(pins: "Pins | None"):
    return ctypes.byref(pins.c) if pins is not None else None


def pins_matrix(ctx: Ctx, g: Csr, part: torch.Tensor, nparts: int, inbound: bool = False) -> Pins:
    """f3: sparse pins(p, e) (inbound=False) or pins_in(p, e) (inbound=True) of part (u32 device)."""
    out = CPins()
    _check(lib().hgp_pins_matrix(ctx.h, ctypes.byref(g.c), _ptr(part), nparts, int(inbound), ctypes.byref(out)))
    return Pins(ctx, out)


def partition_metrics(ctx: Ctx, g: Csr, part: torch.Tensor, nparts: int, omega: int = UNBOUNDED,
                      delta: int = UNBOUNDED, loads: bool = False):
    """f1: Eq.1 connectivity, Eq.16 cut-net, max loads and violation counts of part. With
    loads=True also returns (size [nparts], inbound [nparts]) u64 device tensors."""
    q = CQuality()
    size = inb = None
    if loads:
        size = torch.empty(max(nparts, 1), dtype=torch.uint64, device="cuda")
        inb = torch.empty(max(nparts, 1), dtype=torch.uint64, device="cuda")
    _check(lib().hgp_partition_metrics(ctx.h, ctypes.byref(g.c), _ptr(part), nparts, omega, delta, ctypes.byref(q),
                                       _ptr(size), _ptr(inb)))
    d = {k: int(getattr(q, k)) for k, _ in CQuality._fields_}
    return (d, size, inb) if loads else d


def propose_moves(ctx: Ctx, g: Csr, part: torch.Tensor, nparts: int, omega: int = UNBOUNDED,
                  enforce_size: bool = False, pins: Pins | None = None):
    """f3: Eq.13 proposals -> (dest u32 [N] with NONE = no move, gain i64 [N]) device tensors."""
    dest = torch.empty(max(g.N, 1), dtype=torch.uint32, device="cuda")
    gain = torch.empty(max(g.N, 1), dtype=torch.int64, device="cuda")
    _check(lib().hgp_propose_moves(ctx.h, ctypes.byref(g.c), _ptr(part), nparts, _pins_ref(pins), omega,
                                   int(enforce_size), _ptr(dest), _ptr(gain)))
    return dest[:g.N], gain[:g.N]


def in_sequence_gains(ctx: Ctx, g: Csr, part: torch.Tensor, nparts: int, seq: torch.Tensor, dest: torch.Tensor,
                      pins: Pins | None = None) -> torch.Tensor:
    """f3: Eqs.14-15 in-sequence gains of the moves seq (u32 device) -> i64 [M] device tensor."""
    M = seq.numel()
    out = torch.empty(max(M, 1), dtype=torch.int64, device="cuda")
    _check(lib().hgp_in_sequence_gains(ctx.h, ctypes.byref(g.c), _ptr(part), nparts, _pins_ref(pins), _ptr(seq), M,
                                       _ptr(dest), _ptr(out)))
    return out[:M]


def sequence_violations(ctx: Ctx, g: Csr, part: torch.Tensor, nparts: int, seq: torch.Tensor, dest: torch.Tensor,
                        omega: int, delta: int, pins_in: Pins | None = None) -> torch.Tensor:
    """f4: event-based validation -> violations u32 [M] device tensor."""
    M = seq.numel()
    out = torch.empty(max(M, 1), dtype=torch.uint32, device="cuda")
    _check(lib().hgp_sequence_violations(ctx.h, ctypes.byref(g.c), _ptr(part), nparts, _pins_ref(pins_in), _ptr(seq),
                                         M, _ptr(dest), omega, delta, _ptr(out)))
    return out[:M]


def best_prefix(ctx: Ctx, gain_seq: torch.Tensor, violations: torch.Tensor):
    """f4: the landing point -> (k, best cumulative gain)."""
    k, b = ctypes.c_uint32(), ctypes.c_int64()
    _check(lib().hgp_best_prefix(ctx.h, _ptr(gain_seq), _ptr(violations), gain_seq.numel(), ctypes.byref(k),
                                 ctypes.byref(b)))
    return int(k.value), int(b.value)


# ---- a5 in pieces for node/edge-range shards (include/hgp.h) ----------------------

class Cedges:
    """Pre-merge coarse edges of a fine edge range (library-owned; hgp_cedges_free)."""

    def __init__(self, ctx: Ctx, c: CCedges):
        self.ctx, self.c = ctx, c

    K = property(lambda s: s.c.K)
    P = property(lambda s: s.c.P)

    def tensors(self) -> dict:
        c = self.c
        return {"eid": dev_view(c.eid, c.K, "u32", self), "fp": dev_view(c.fp, c.K, "u64", self),
                "nsrc": dev_view(c.nsrc, c.K, "u32", self), "size": dev_view(c.size, c.K, "u32", self),
                "off": dev_view(c.off, c.K + 1, "u64", self), "pins": dev_view(c.pins, c.P, "u32", self)}

    def free(self):
        if self.c is not None and self.ctx.h:
            lib().hgp_cedges_free(self.ctx.h, ctypes.byref(self.c))
        self.c = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class CedgesView:
    """hgp_cedges over torch-owned device tensors (e.g. the all-gathered ranges)."""

    def __init__(self, eid, fp, nsrc, size, off, pins):
        self.t = [x.contiguous() for x in (eid, fp, nsrc, size, off, pins)]
        K = self.t[0].numel()
        self.c = CCedges(K, 0, self.t[5].numel(), *[vp(x.data_ptr()) for x in self.t])


def gamma(ctx: Ctx, match_t: torch.Tensor, N: int, out: torch.Tensor) -> int:
    """hgp_gamma: coarse ids of a symmetric match into out (u32 [N]); returns N'."""
    nc = ctypes.c_uint32()
    _check(lib().hgp_gamma(ctx.h, _ptr(match_t), N, _ptr(out), ctypes.byref(nc)))
    return nc.value


def coarse_bounds(ctx: Ctx, match_t: torch.Tensor, N: int, bounds: list[int]) -> list[int]:
    arr_in = (ctypes.c_uint32 * len(bounds))(*bounds)
    arr_out = (ctypes.c_uint32 * len(bounds))()
    _check(lib().hgp_coarse_bounds(ctx.h, _ptr(match_t), N, arr_in, len(bounds), arr_out))
    return list(arr_out)


def contract_edges(ctx: Ctx, g: Csr, gamma_t: torch.Tensor, elo: int, ehi: int) -> Cedges:
    out = CCedges()
    _check(lib().hgp_contract_edges(ctx.h, ctypes.byref(g.c), _ptr(gamma_t), elo, ehi, ctypes.byref(out)))
    return Cedges(ctx, out)


def contract_merge(ctx: Ctx, g: Csr, match_t: torch.Tensor, gamma_t: torch.Tensor, allv: CedgesView) -> Csr:
    out = CCsr()
    _check(lib().hgp_contract_merge(ctx.h, ctypes.byref(g.c), _ptr(match_t), _ptr(gamma_t), ctypes.byref(allv.c),
                                    ctypes.byref(out)))
    return Csr(ctx, out)


def coarse_neighbors(ctx: Ctx, match_t: torch.Tensor, gamma_t: torch.Tensor, N: int, seg_start: torch.Tensor,
                     seg_len: torch.Tensor, nbr: torch.Tensor, clo: int, chi: int) -> Nbrs:
    out = CNbrs()
    _check(lib().hgp_coarse_neighbors(ctx.h, _ptr(match_t), _ptr(gamma_t), N, _ptr(seg_start), _ptr(seg_len), _ptr(nbr),
                                      clo, chi, ctypes.byref(out)))
    return Nbrs(ctx, out)
