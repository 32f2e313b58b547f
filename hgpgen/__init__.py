"""hgpgen — seeded synthetic inputs shared by the oracle tests and the CUDA path.

Only inputs live here (hypergraphs + the workload's parameter values); none of
the coarsening arithmetic does.  The C generator (hgpgen.c) is compiled to
``hgpgen/libhgpgen.so`` by ``__graft_entry__.build()`` / ``make``.

Workloads follow SURVEY.md §8(d) / BASELINE.json ``configs``:
  C1 tiny, C2 SNN-1M (-model / -rand), C3 VLSI-like power law, C4 k-way k=2,
  C5 billion-pin SNN.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

UNBOUNDED = (1 << 64) - 1


class _Graph(ctypes.Structure):
    _fields_ = [
        ("num_nodes", ctypes.c_uint32),
        ("num_edges", ctypes.c_uint32),
        ("num_pins", ctypes.c_uint64),
        ("edge_off", ctypes.POINTER(ctypes.c_uint64)),
        ("edge_nsrc", ctypes.POINTER(ctypes.c_uint32)),
        ("pins", ctypes.POINTER(ctypes.c_uint32)),
        ("edge_w", ctypes.POINTER(ctypes.c_uint32)),
        ("node_w", ctypes.POINTER(ctypes.c_uint32)),
    ]


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libhgpgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} gen`")
        lib = ctypes.CDLL(path)
        G = ctypes.POINTER(_Graph)
        u32, u64, dbl = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
        lib.hgpgen_tiny.argtypes = [u64, u32, u32, u32, u32, u32, u32, u32, G]
        lib.hgpgen_snn.argtypes = [u64, u32, u32, u32, u32, u32, dbl, G]
        lib.hgpgen_vlsi.argtypes = [u64, u32, u32, u32, u32, dbl, dbl, u32, G]
        for f in (lib.hgpgen_tiny, lib.hgpgen_snn, lib.hgpgen_vlsi):
            f.restype = ctypes.c_int
        lib.hgpgen_free.argtypes = [G]
        lib.hgpgen_free.restype = None
        _LIB = lib
    return _LIB


@dataclass
class Hypergraph:
    """Host copy of a generated problem statement."""

    num_nodes: int
    edge_off: np.ndarray   # u64 [E+1]
    edge_nsrc: np.ndarray  # u32 [E]
    pins: np.ndarray       # u32 [P]
    edge_w: np.ndarray     # u32 [E]
    node_w: np.ndarray     # u32 [N]
    name: str = ""

    @property
    def num_edges(self) -> int:
        return int(self.edge_nsrc.shape[0])

    @property
    def num_pins(self) -> int:
        return int(self.pins.shape[0])

    def input_bytes(self) -> int:
        return sum(a.nbytes for a in (self.edge_off, self.edge_nsrc, self.pins, self.edge_w, self.node_w))


def _take(g: _Graph, name: str) -> Hypergraph:
    N, E, P = g.num_nodes, g.num_edges, g.num_pins

    def arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dtype=dt)
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

    hg = Hypergraph(
        num_nodes=N,
        edge_off=arr(g.edge_off, E + 1, np.uint64),
        edge_nsrc=arr(g.edge_nsrc, E, np.uint32),
        pins=arr(g.pins, P, np.uint32),
        edge_w=arr(g.edge_w, E, np.uint32),
        node_w=arr(g.node_w, N, np.uint32),
        name=name,
    )
    _lib().hgpgen_free(ctypes.byref(g))
    return hg


def tiny(seed: int, num_nodes: int = 1000, num_edges: int = 3000, size_base: int = 2,
         size_binom: int = 12, in_cap: int = 32, wmax_e: int = 8, wmax_n: int = 1) -> Hypergraph:
    g = _Graph()
    rc = _lib().hgpgen_tiny(seed, num_nodes, num_edges, size_base, size_binom, in_cap, wmax_e,
                            wmax_n, ctypes.byref(g))
    if rc != 0:
        raise ValueError("hgpgen_tiny failed")
    return _take(g, f"tiny(seed={seed},N={num_nodes},E={num_edges})")


def snn(seed: int, layers: int = 10, rows: int = 250, cols: int = 400, fanout: int = 99,
        window: int = 15, rewire: float = 0.0) -> Hypergraph:
    g = _Graph()
    rc = _lib().hgpgen_snn(seed, layers, rows, cols, fanout, window, rewire, ctypes.byref(g))
    if rc != 0:
        raise ValueError("hgpgen_snn failed")
    kind = "rand" if rewire > 0 else "model"
    return _take(g, f"snn-{kind}(seed={seed},{layers}x{rows}x{cols},F={fanout})")


def vlsi(seed: int, num_nodes: int = 5_000_000, num_edges: int = 5_000_000, dmin: int = 2,
         dmax: int = 1024, alpha: float = 2.005, locality: float = 0.9,
         in_cap: int = 4096) -> Hypergraph:
    g = _Graph()
    rc = _lib().hgpgen_vlsi(seed, num_nodes, num_edges, dmin, dmax, alpha, locality, in_cap,
                            ctypes.byref(g))
    if rc != 0:
        raise ValueError("hgpgen_vlsi failed")
    return _take(g, f"vlsi(seed={seed},N={num_nodes},E={num_edges})")


@dataclass
class Workload:
    """A BASELINE.json config: the hypergraph recipe plus the level's parameters."""

    name: str
    make: object                 # callable(seed) -> Hypergraph
    omega: int                   # size limit Omega
    delta: int                   # inbound limit Delta; UNBOUNDED = +inf
    pi: int = 4                  # candidates per node
    noise: bool = True
    extra: dict = field(default_factory=dict)


def default_noise_cap(hg: Hypergraph) -> int:
    """Config default for the noise cap: floor(0.1 * mean_e omega(e) * 2^24)
    ("caps at 10% of mean h-edge weight"; reading #3)."""
    if hg.num_edges == 0:
        return 0
    return int((int(hg.edge_w.astype(np.uint64).sum()) << 24) // (10 * hg.num_edges))


def kway_omega(hg: Hypergraph, k: int = 2, eps: float = 0.03) -> int:
    """Omega = floor((1+eps) * W / k)."""
    W = int(hg.node_w.astype(np.uint64).sum())
    return int((1.0 + eps) * W / k)


WORKLOADS = {
    "C1": Workload("C1 tiny", lambda s: tiny(s), 16, 32),
    "C2": Workload("C2 SNN-1M-model", lambda s: snn(s), 256, 4096),
    "C2r": Workload("C2 SNN-1M-rand", lambda s: snn(s, rewire=0.1), 256, 4096),
    "C3": Workload("C3 VLSI-5M", lambda s: vlsi(s), 256, 4096),
    "C4": Workload("C4 k-way k=2 (1M nodes)", lambda s: vlsi(s, 1_000_000, 1_000_000), -1, UNBOUNDED,
                   extra={"kway": 2}),
    "C5": Workload("C5 SNN-10M (1e9 pins)", lambda s: snn(s, rows=1000, cols=1000), 256, 4096),
}
