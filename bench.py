#!/usr/bin/env python
"""bench.py — throughput of one coarsening level of arXiv 2605.20497 on B200.

Metric (BASELINE.json): pins processed per second per coarsening level. One "step" is
one pass of the whole hot path over one synthetic input:
    a1 hgp_build_csr -> a2 hgp_unique_neighbors -> hgp_coarsen_level (a3 score, a4 match, a5 contract)
on the level-0 hypergraph of the configured workload (default C2: SNN-mapping, 1M neurons,
1e8 pins, Omega=256, Delta=4096, Pi=4, noise on).

  value : P / device time of the step (inputs resident in HBM; CUDA events, max over ranks)
  e2e   : the same through the C-ABI with HOST inputs: per step the pinned-host -> device copy
          of the input arrays and the device -> host read of gamma are inside the timed region
  roofline: the dominant kernel's algorithmic bytes / its live CUDA-event
          time over the timed region, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline: the CPU oracle (oracle/, single thread) on a bounded sample of the same recipe

`--impl reference` times the oracle alone (the tier's reference arm) on a bounded sample.
Multi-GPU (torchrun, N>1): the level is sharded (shard.py): every rank holds the
replicated CSR, runs the fused a2+a3 on its equal-work node range; the candidate rows are
all-gathered (NCCL), a4 runs replicated, a5 builds the coarse edges of the rank's edge range, the
ranges are all-gathered and merged replicated, and each rank builds the coarse neighbours of its
coarse node range with a halo exchange of partners' N(b). value = P / step time (strong scaling;
bit-identical to 1 GPU). The line carries the per-phase compute / communication split.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

# Library arrays come from torch's caching allocator; expandable segments keep the level's
# tens-of-GB buffers (C5: the 2^34-entry neighbour pool, the coarse-neighbour bound pool) from
# fragmenting its cache across steps.
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hgpgen  # noqa: E402

METRIC = "pins/sec per coarsening level (a1..a5 on level 0)"
UNIT = "pins/s"


def _workload(name: str, seed: int):
    w = hgpgen.WORKLOADS[name]
    hg = w.make(seed)
    omega = w.omega if w.omega > 0 else hgpgen.kway_omega(hg, w.extra.get("kway", 2))
    cap = hgpgen.default_noise_cap(hg) if w.noise else 0
    return w, hg, omega, w.delta, w.pi, cap


def algorithmic_bytes(step: str, N, E, P, V, pi, Nc=0, Ec=0, Pc=0, Vc=0) -> int:
    """Minimum bytes each step must move (every array element read once, every output written
    once; gathers counted once per element) — SURVEY §8(d), restated in DESIGN.md §Roofline."""
    if step == "a1":
        return 12 * P + 36 * E + 24 * N
    if step == "a2":
        return 8 * P + 8 * E + 16 * N + 4 * V
    if step == "a3":
        return 4 * V + 8 * P + 20 * E + 28 * N + 16 * pi * N
    if step == "a4":
        return 16 * pi * N + 4 * N
    if step == "a2+a3":   # the fused kernel does both rows: charged their sum
        return algorithmic_bytes("a2", N, E, P, V, pi) + algorithmic_bytes("a3", N, E, P, V, pi)
    if step == "a5":
        return 16 * N + 4 * P + 20 * E + 8 * Pc + 20 * Ec + 4 * V + 4 * Vc + 28 * Nc
    raise KeyError(step)


KERNEL_STEP = {"nbrscore": "a2+a3", "hub_": "a2+a3", "small_split": "a2+a3", "pairs_total": "a2+a3", "fused_pack": "a2+a3", "validate": "a1", "check": "a1", "segsort": "a1", "inc_": "a1", "fill_mu": "a1", "max_deg": "a1",
               "radix_": "a1", "edge_pairs": "a2", "nbrs_": "a2", "nbr_": "a2", "score_": "a3", "round_": "a4", "jump_": "a4",
               "fill_none": "a4"}


def step_of(kernel: str) -> str:
    for k, v in KERNEL_STEP.items():
        if kernel.startswith(k):
            return v
    return "a5"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        loaded = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_record(kernel: str, workload: str) -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    return json.load(open(p)).get(workload, {}).get(kernel) or {}


def ncu_traffic(kernel: str, workload: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    rec = d.get(workload, {}).get(kernel)
    return rec.get("dram_bytes_per_launch") if rec else None


# ------------------------------------------------------------------------------------------ oracle legs
def oracle_level_seconds(hg, omega, delta, pi, cap, seed) -> float:
    from oracle import ref
    t0 = time.perf_counter()
    g = ref.build_csr_hg(hg)
    nb = ref.unique_neighbors(g)
    ref.coarsen_level(g, nb, ref.params(omega, delta, pi, noise_seed=seed, noise_cap=cap))
    return time.perf_counter() - t0


def oracle_sample(workload: str, seed: int, scale: str):
    """A bounded sample of the workload's recipe for the single-threaded oracle."""
    if workload.startswith("C2") or workload == "C5":
        rows, cols = (50, 80) if scale == "baseline" else (25, 40)
        rew = 0.1 if workload == "C2r" else 0.0
        hg = hgpgen.snn(seed, rows=rows, cols=cols, rewire=rew)
        desc = f"SNN recipe (C2 generator) at 10 layers x {rows}x{cols} = {10 * rows * cols} neurons, " \
               f"{hg.num_pins} pins; full level a1..a5"
        return hg, 256, 4096, desc
    n = 400_000 if scale == "baseline" else 100_000
    hg = hgpgen.vlsi(seed, n, n)
    om = 256 if workload == "C3" else hgpgen.kway_omega(hg)
    de = 4096 if workload == "C3" else hgpgen.UNBOUNDED
    return hg, om, de, f"VLSI recipe at {n} nodes/edges, {hg.num_pins} pins; full level a1..a5"


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    hg, om, de, desc = oracle_sample(args.workload, args.seed, "reference")
    cap = hgpgen.default_noise_cap(hg)
    for _ in range(args.warmup):
        oracle_level_seconds(hg, om, de, 4, cap, args.seed)
    ts = [oracle_level_seconds(hg, om, de, 4, cap, args.seed) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    value = hg.num_pins / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64", "data": "synthetic",
            "config": {"workload": hgpgen.WORKLOADS[args.workload].name, "sample": desc},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pin_visits(edge_off: np.ndarray) -> int:
    """T = sum over e of |e| (|e| - 1): the pin visits of a2/a3's traversal (SURVEY §8 symbols)."""
    d = np.diff(edge_off.astype(np.int64))
    return int((d * (d - 1)).sum())


def smem_roofline(visits_per_launch: float, ms_per_launch: float, clk: dict):
    """The shared-memory roofline of the traversal: every pin visit needs at least
    one 4-byte key load and one 4-byte atomic add in shared memory, 8 B through the 128 B/cycle/SM
    crossbar (B300_MICROARCH "LDS/STS": 128/N B/cyc/SM, N = 1 without bank conflicts), so at most
    16 visits per cycle per SM."""
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak = 16.0 * sms * mhz * 1e6
    achieved = visits_per_launch / (ms_per_launch * 1e-3)
    return achieved, peak, f"128 B/cycle/SM smem crossbar / 8 B per visit x {sms} SMs x {mhz:.0f} MHz (sampled)"


def issue_roofline(kernel: str, workload: str, ms_per_launch: float, clk: dict):
    """The dominant kernel is bound by instruction issue, not HBM: its warp-
    instruction count per launch (committed ncu capture) over its live CUDA-event time, against
    4 warp-instructions / cycle / SM x SMs x the SM clock sampled during the timed region."""
    rec = ncu_record(kernel, workload)
    wi = rec.get("warp_instructions")
    if not wi or not ms_per_launch:
        return None
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak = 4.0 * sms * mhz * 1e6
    achieved = wi / (ms_per_launch * 1e-3)
    return {"unit": "warp-instructions/s", "achieved": achieved, "peak": peak,
            "frac": achieved / peak, "warp_instructions_per_launch": wi,
            "peak_derivation": f"4 issue slots/cycle/SM x {sms} SMs x {mhz:.0f} MHz (sampled)"}


def refine_leg(hgp, ctx, hierarchy, omega, delta, stream):
    """SURVEY §8(f) on the bench input: f1 = Eq.1 / Eq.16 / loads of the initial partition rho of the
    hierarchy on level 0; f3 + f4 = one refinement step on it, each call timed with CUDA
    events: pins and pins_in matrices, Eq.13 proposals (size-enforcing), in-sequence
    gains, event-based violations and the landing point. The move sequence is the proposals in
    gain order (built untimed; the chaining of P:944-960 is not one of these rows). Applying the
    landing prefix and re-measuring Eq.1 checks the whole step: Eq.1 must drop by exactly `best`."""
    import torch
    _, _, g, rho, cg = hierarchy(keep=True)
    nparts = cg.N
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t = {}

    def timed(name, fn):
        a, b = ev(), ev()
        a.record(stream)
        out = fn()
        b.record(stream)
        torch.cuda.synchronize()
        t[name] = round(a.elapsed_time(b), 3)
        return out

    q = timed("f1_quality", lambda: hgp.partition_metrics(ctx, g, rho, nparts, omega, delta))
    pins = timed("pins", lambda: hgp.pins_matrix(ctx, g, rho, nparts))
    pins_in = timed("pins_in", lambda: hgp.pins_matrix(ctx, g, rho, nparts, inbound=True))
    dest, gain = timed("propose_moves", lambda: hgp.propose_moves(ctx, g, rho, nparts, omega, True, pins=pins))
    movers = torch.nonzero(dest.view(torch.int32) != -1).flatten()       # dest != NONE
    order = torch.argsort(-gain[movers], stable=True)
    seq = movers[order].to(torch.int32).contiguous()                     # u32 ids (int32 view)
    gs = timed("in_sequence_gains", lambda: hgp.in_sequence_gains(ctx, g, rho, nparts, seq, dest, pins=pins))
    vio = timed("sequence_violations",
                lambda: hgp.sequence_violations(ctx, g, rho, nparts, seq, dest, omega, delta, pins_in=pins_in))
    k, best = timed("best_prefix", lambda: hgp.best_prefix(ctx, gs, vio))
    moved = rho.view(torch.int32).clone()
    if k:
        idx = seq[:k].long()
        moved[idx] = dest.view(torch.int32)[idx]
    q2 = hgp.partition_metrics(ctx, g, moved, nparts, omega, delta)
    for x in (pins, pins_in, g, cg):
        x.free()
    out = {"what": "one refinement step on rho (f3 Eq.13 + Eqs.14-15, f4 P:1032-1057), GPU calls timed",
           "nparts": nparts, "moves_proposed": int(seq.numel()), "landing_prefix": k, "gain": best,
           "connectivity_before": q["connectivity"], "connectivity_after": q2["connectivity"],
           "gain_checks": q["connectivity"] - q2["connectivity"] == best,
           "violations_after": q2["size_violations"] + q2["inbound_violations"], "ms": t,
           "total_ms": round(sum(t.values()), 3)}
    return q, out


# ------------------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hgp", choices=["hgp", "reference"])
    ap.add_argument("--workload", default="C2", choices=sorted(hgpgen.WORKLOADS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-refine", action="store_true", help="skip the f1 quality / f3-f4 refinement-step leg")
    ap.add_argument("--no-hier", action="store_true", help="skip the whole-hierarchy leg (implies --no-refine)")
    ap.add_argument("--dominant", default=None, help="kernel name for the roofline (default: measured top kernel)")
    ap.add_argument("--share-device", action="store_true",
                    help="testing the N>1 code path on one GPU: every rank on cuda:0, gloo instead of NCCL")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2605_20497_b200 import hgp

    assert args.warmup >= 3 or os.environ.get("HGP_BENCH_ALLOW_SHORT"), "timing rules need >= 3 warm-up steps"
    if args.share_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w, hg, omega, delta, pi, cap = _workload(args.workload, args.seed)
    N, E, P = hg.num_nodes, hg.num_edges, hg.num_pins
    stream = torch.cuda.current_stream()
    ctx = hgp.Ctx(local, stream=stream)
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(hg, k))).pin_memory()
            for k in ("edge_off", "edge_nsrc", "pins", "edge_w", "node_w")}
    dev = {k: v.cuda() for k, v in host.items()}
    h2d_bytes = sum(v.numel() * v.element_size() for v in host.values())
    params = hgp.params(omega, delta, pi, noise_seed=args.seed, noise_cap=cap)
    cand = hgp.empty_cand(N, pi)
    match = torch.empty(N, dtype=torch.uint32, device="cuda")
    gamma = torch.empty(N, dtype=torch.uint32, device="cuda")
    gamma_host = torch.empty(N, dtype=torch.uint32).pin_memory()

    last = {}

    from paper_2605_20497_b200 import shard
    comm = shard.DistComm() if world > 1 else None

    def step(inp):
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        g = hgp.build_csr(ctx, N, inp["edge_off"], inp["edge_nsrc"], inp["pins"], inp["edge_w"], inp["node_w"])
        eb.record(stream)
        last["a1_events"] = (ea, eb)
        if world == 1:   # N(n) is consumed by a5 where the fused kernel left it (not returned)
            nb, cg, cnb, st = hgp.coarsen_level0(ctx, g, params, cand, match, gamma, want_nbrs=False)
        else:   # the sharded level (shard.py): a2+a3 / a5 on this rank's ranges, NCCL exchanges
            bounds = hgp.shard_bounds(ctx, g, world)
            states = [shard.RankState(rank, bounds[rank], bounds[rank + 1])]
            cg, info = shard.level_sharded(ctx, g, params, states, comm, True, cand, match, gamma)
            cnb, nb = states[0].nb, None
            vt = torch.tensor([info.V, cnb.V], dtype=torch.int64, device="cpu" if args.share_device else "cuda")
            dist.all_reduce(vt)                                          # V and V' summed over the ranks
            st = {"Nc": cg.N, "Ec": cg.E, "Pc": cg.P, "Vc": int(vt[1].item()), "V": int(vt[0].item()),
                  "matched_per_round": [info.pairs],
                  "purged": 0, "merged_edges": 0, "dropped_edges": 0, "phase_ms": info.ms}
        last.update(st=st, V=nb.V if nb is not None else st["V"])
        for x in (g, nb, cg, cnb):
            if x is not None:
                x.free()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.share_device else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step(dev)
    torch.cuda.synchronize()

    # ---- per-kernel breakdown (one untimed, profiled step) -> dominant kernel
    ctx.profile_begin("")
    step(dev)
    ctx.profile_end()
    breakdown = ctx.profile_report()
    dominant = args.dominant or max(breakdown, key=lambda k: breakdown[k][0])
    # the dominant kernel's family (every tier launch of it in a step, e.g. nbrscore_S/A/M/B):
    # the step's algorithmic work is charged to their summed device time
    family = dominant.rsplit("_", 1)[0] if dominant.split("_")[-1] in ("S", "A", "M", "B", "W", "H", "C", "A2") else dominant

    # ---- timed region: K steps, inputs resident in HBM (420 MB > 126 MB L2)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    l0 = ctx.launches
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile_begin(family)
    ev0.record(stream)
    for _ in range(args.steps):
        step(dev)
    ev1.record(stream)
    torch.cuda.synchronize()
    dom_ms, dom_launches = ctx.profile_end()
    barrier()
    launches = ctx.launches - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    clk = clocks.stop()

    # ---- end-to-end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        bufs = {k: torch.empty_like(v) for k, v in dev.items()}

        def step_e2e():
            for k in bufs:
                ctx.copy(bufs[k].data_ptr(), host[k].data_ptr(), host[k].numel() * host[k].element_size())
            step(bufs)
            ctx.copy(gamma_host.data_ptr(), gamma.data_ptr(), 4 * N)

        step_e2e()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_e2e()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        e2e = {"value": P / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": 4 * N}

    # ---- whole hierarchy: a1 + hgp_coarsen to the stop rule, 1 GPU, CUDA events
    hier = None
    refine = None
    if args.no_hier:
        pass
    elif world == 1:
        def hierarchy(keep=False):
            g = hgp.build_csr(ctx, N, dev["edge_off"], dev["edge_nsrc"], dev["pins"], dev["edge_w"], dev["node_w"])
            rho, cg, cnb, levels = hgp.coarsen(ctx, g, params)
            out = (levels, cg.N)
            if keep:
                cnb.free()
                return out + (g, rho, cg)
            for x in (g, cg, cnb):
                x.free()
            return out
        hierarchy()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        levels, n_last = hierarchy()
        h1.record(stream)
        torch.cuda.synchronize()
        hms = h0.elapsed_time(h1)
        hier = {"what": "a1 + every level to the stop rule (hgp_coarsen, reading #21)", "levels": len(levels),
                "total_coarsening_ms": hms, "pins_per_s": P / (hms / 1e3), "coarsest_nodes": n_last,
                "level_ms": [round(l["ms"]["total"], 3) for l in levels],
                "level_nodes": [l["N"] for l in levels],
                "matched_fraction": [round(2 * sum(l["matched_per_round"]) / max(l["N"], 1), 4) for l in levels]}
        # the same hierarchy with f2 (leftover pairing, HGP_FLAG_LEFTOVER): how close the stop
        # rule's ceil(W / Omega) gets
        pf2 = hgp.params(omega, delta, pi, noise_seed=args.seed, noise_cap=cap, flags=hgp.FLAG_LEFTOVER)
        g2 = hgp.build_csr(ctx, N, dev["edge_off"], dev["edge_nsrc"], dev["pins"], dev["edge_w"], dev["node_w"])
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        _, cg2, cnb2, lv2 = hgp.coarsen(ctx, g2, pf2)
        f1.record(stream)
        torch.cuda.synchronize()
        Wt = int(hg.node_w.astype(np.int64).sum())
        hier["with_f2"] = {"levels": len(lv2), "coarsest_nodes": cg2.N, "total_coarsening_ms": f0.elapsed_time(f1),
                           "stop_target_ceil_W_over_omega": -(-Wt // omega) if omega < hgpgen.UNBOUNDED else 1}
        hier["stop_target_ceil_W_over_omega"] = hier["with_f2"]["stop_target_ceil_W_over_omega"]
        for x in (g2, cg2, cnb2):
            x.free()
        if not args.no_refine:
            try:
                hier_q, refine = refine_leg(hgp, ctx, hierarchy, omega, delta, stream)
                hier["initial_partition"] = hier_q
            except hgp.HgpError as ex:   # an optional leg: its status is reported, the line stands
                # (e.g. C5: more than 2^29 inbound events for f4's 32-bit event keys -> HGP_E_OVERFLOW)
                refine = {"error": str(ex)}
                torch.cuda.synchronize()
    else:   # the sharded driver (shard.coarsen_sharded): same levels as hgp_coarsen, per-phase split
        def hierarchy_sharded():
            g = hgp.build_csr(ctx, N, dev["edge_off"], dev["edge_nsrc"], dev["pins"], dev["edge_w"], dev["node_w"])
            rho, levels, cg, states = shard.coarsen_sharded(ctx, g, params, comm)
            n_last = cg.N
            for x in [g, cg] + [s_.nb for s_ in states]:
                x.free()
            return levels, n_last
        hierarchy_sharded()
        barrier()
        t_0 = time.perf_counter()
        levels, n_last = hierarchy_sharded()
        torch.cuda.synchronize()
        hms = max_over_ranks((time.perf_counter() - t_0) * 1e3)
        phases = {}
        for l in levels:
            for k, v in l.ms.items():
                phases[k] = round(phases.get(k, 0.0) + v, 3)
        comm_ms = sum(v for k, v in phases.items() if k.startswith("X"))
        hier = {"what": "a1 + every level to the stop rule, sharded (shard.coarsen_sharded; host wall clock, max "
                        "over ranks)", "levels": len(levels), "total_coarsening_ms": hms, "pins_per_s": P / (hms / 1e3),
                "coarsest_nodes": n_last, "level_nodes": [l.N for l in levels], "phase_ms_total": phases,
                "comm_ms": round(comm_ms, 3), "compute_ms": round(sum(phases.values()) - comm_ms, 3)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    st = last["st"]
    V = last["V"]
    dstep = step_of(dominant)
    alg = algorithmic_bytes(dstep, N, E, P, V, pi, st["Nc"], st["Ec"], st["Pc"], st["Vc"])
    fam_ms_step = dom_ms / args.steps                       # the family's device time per step
    achieved = alg / (fam_ms_step * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    rec = ncu_record(dominant, args.workload)
    hbm_view = {"achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "alg_bytes_per_step": alg, "traffic": rec.get("dram_bytes_per_launch")}
    roof = {"bound": "hbm", **hbm_view}
    if dstep in ("a2+a3", "a3", "a2"):
        # measured: the traversal kernels use a few % of DRAM bandwidth and most issue slots
        # (profiles/ncu_traffic.json), so the binding roofline is the shared-memory visit rate
        T = pin_visits(hg.edge_off)
        va, vp, deriv = smem_roofline(T, fam_ms_step, clk)
        measured_bound = "alu" if (rec.get("issue_pct") or 100.0) > (rec.get("dram_pct") or 0.0) else "hbm"
        if measured_bound == "alu":
            roof = {"bound": "alu", "achieved": va, "peak": vp, "unit": "pin-visits/s", "frac": va / vp,
                    "visits_per_step": T, "peak_derivation": deriv, "traffic": rec.get("dram_bytes_per_launch"),
                    "hbm": hbm_view}
    roof.update({"kernel": dominant, "family": family, "step": dstep, "ms_per_step": fam_ms_step,
                 "launches_per_step": dom_launches / args.steps,
                 "ncu": {k: rec.get(k) for k in ("dram_pct", "issue_pct", "l2_hit_pct", "ipc_active")} if rec else None})
    # per step of the path from CUDA events around the API calls of the last step (a1 = hgp_build_csr;
    # a2+a3 / a4 / a5 = the level's own events, hgp_level_stats.ms), not from kernel-name guesses
    ea, eb = last["a1_events"]
    step_ms = {"a1": ea.elapsed_time(eb)}
    if isinstance(st.get("ms"), dict):
        step_ms.update({"a2+a3": st["ms"]["score"], "a4": st["ms"]["match"], "a5": st["ms"]["contract"]})
    line = {
        "metric": METRIC, "value": P / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "u32/u64 (integer fixed point)", "data": "synthetic",
        "config": {"workload": w.name, "N": N, "E": E, "P": P, "V": V, "omega": omega,
                   "delta": "inf" if delta == hgpgen.UNBOUNDED else delta, "pi": pi, "noise_cap": cap,
                   "seed": args.seed,
                   "parallelism": "1 GPU" if world == 1 else
                   f"{world} ranks: a2+a3 on node ranges, a5 edges on edge ranges, a5 N' on coarse node ranges; "
                   f"X1 cand all-gather, X2 pre-merge coarse-edge all-gather, X3 halo send/recv (NCCL); a1, a4 and "
                   f"the merge replicated",
                   "l2": "inputs (%.0f MB) larger than L2" % (h2d_bytes / 1e6)},
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roof,
        "issue_roofline": issue_roofline(dominant, args.workload, fam_ms_step, clk),
        "level": {"Nc": st["Nc"], "Ec": st["Ec"], "Pc": st["Pc"], "Vc": st["Vc"], "phase_ms": st.get("phase_ms"),
                  "matched_fraction": float((match.view(torch.int32) != -1).sum().item()) / N,
                  "matched_per_round": st["matched_per_round"], "purged": st["purged"],
                  "merged_edges": st["merged_edges"], "dropped_edges": st["dropped_edges"]},
        "step_ms": {k: round(v, 4) for k, v in sorted(step_ms.items())},
        "kernels_ms": {k: round(v[0], 4) for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1][0])[:12]},
        "level_hbm_frac": sum(algorithmic_bytes(s, N, E, P, V, pi, st["Nc"], st["Ec"], st["Pc"], st["Vc"])
                              for s in ("a1", "a2+a3", "a4", "a5")) / (ms * 1e-3) / 1e9 / peak,
    }
    if e2e:
        line["e2e"] = e2e
    if hier:
        line["hierarchy"] = hier
    if refine:
        line["refine_step"] = refine
    if world == 1 and not args.no_cpu_baseline:
        hs, om, de, desc = oracle_sample(args.workload, args.seed, "baseline")
        t = oracle_level_seconds(hs, om, de, pi, hgpgen.default_noise_cap(hs), args.seed)
        line["cpu_baseline"] = {"value": hs.num_pins / t, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": desc, "seconds": t, "host_cores": os.cpu_count()}
        gold = os.path.join(ROOT, "tests", "golden", f"{args.workload}_s{args.seed}.json")
        if os.path.exists(gold):   # the oracle on the FULL input (tools/golden_full.py; recorded, not re-run)
            gd = json.load(open(gold))
            if "oracle_seconds" in gd:
                line["cpu_baseline"]["full_input"] = {
                    "value": gd["oracle_pins_per_s"], "unit": UNIT, "seconds": gd["oracle_seconds"]["total"],
                    "cores": gd.get("oracle_host", {}).get("cores_used", 1),
                    "where": "build container, tools/golden_full.py (recorded)", "per_step_s": gd["oracle_seconds"]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
