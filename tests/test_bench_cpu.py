"""Host logic of bench.py (CPU): the algorithmic-byte model of DESIGN.md §5, the kernel -> step
attribution, and the reference arm's JSON contract (the oracle on a bounded sample)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_algorithmic_bytes_model():
    N, E, P, V, pi = 10 ** 6, 10 ** 6, 10 ** 8, 963651260, 4
    # the fused a2+a3 kernel is charged both rows (16P + 28E + 44N + 8V + 16 pi N)
    assert bench.algorithmic_bytes("a2+a3", N, E, P, V, pi) == 16 * P + 28 * E + 44 * N + 8 * V + 16 * pi * N
    assert bench.algorithmic_bytes("a1", N, E, P, V, pi) == 12 * P + 36 * E + 24 * N
    assert bench.algorithmic_bytes("a4", N, E, P, V, pi) == 16 * pi * N + 4 * N
    Nc, Ec, Pc, Vc = 586685, 10 ** 6, 81582221, 413518770
    assert bench.algorithmic_bytes("a5", N, E, P, V, pi, Nc, Ec, Pc, Vc) == \
        16 * N + 4 * P + 20 * E + 8 * Pc + 20 * Ec + 4 * V + 4 * Vc + 28 * Nc


def test_pin_visits():
    import numpy as np
    off = np.array([0, 3, 4, 104], dtype=np.uint64)          # |e| = 3, 1, 100
    assert bench.pin_visits(off) == 3 * 2 + 0 + 100 * 99


def test_kernel_step_attribution():
    assert bench.step_of("nbrscore_A") == "a2+a3" and bench.step_of("nbrscore_S") == "a2+a3"
    assert bench.step_of("score_F") == "a3" and bench.step_of("round_up") == "a4"
    assert bench.step_of("inc_count") == "a1" and bench.step_of("coarse_nbrs_A") == "a5"


def test_reference_arm_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "pins/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["workload"].startswith("C2")
