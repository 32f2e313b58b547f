"""CPU-side checks of the C-ABI library: it loads and exports every symbol include/hgp.h declares
(no compute calls — there is no GPU here), and the product binding has no CPU fallback."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_20497_b200", "libhgp.so")


def declared():
    hdr = open(os.path.join(ROOT, "include", "hgp.h")).read()
    return sorted(set(re.findall(r"HGP_API\s+[\w\s\*]+?\b(hgp_\w+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", ROOT, "cuda"], check=True)
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_entry_points():
    names = declared()
    for n in ("hgp_build_csr", "hgp_unique_neighbors", "hgp_score_pairs", "hgp_match", "hgp_contract",
              "hgp_coarsen_level"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in declared():
        assert hasattr(lib, n), n


def test_exports_are_only_the_abi(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = sorted({l.split()[-1] for l in out.splitlines() if " T " in l and l.split()[-1].startswith("hgp_")})
    assert exported == declared()


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_80" not in out and "sm_90" not in out


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_20497_b200 import hgp
    with pytest.raises(RuntimeError):
        hgp.Ctx(0)


def test_product_never_imports_the_oracle():
    pat = re.compile(r"(import\s+oracle|from\s+oracle|hgp_ref|libhgp_ref)")
    pkg = os.path.join(ROOT, "paper_2605_20497_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                assert not pat.search(open(os.path.join(dp, f)).read()), f
    out = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "hgp_ref" not in out
