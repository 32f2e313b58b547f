"""Per-source-line instruction counts and stall samples for one kernel of an .ncu-rep.
Joins ncu's per-SASS-instruction metrics with nvdisasm -g line info of the library cubins.
usage: python tools/ncu_lines.py REP KERNEL_REGEX MANGLED_NAME [top]"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(mangled):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2605_20497_b200", "libhgp.so")],
                   cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        sec = out.find(f".text.{mangled}:")
        if sec < 0:
            continue
        body = out[sec:]
        end = body.find("//---------------------", 10)
        body = body[:end] if end > 0 else body
        cur = None
        m = {}
        for ln in body.splitlines():
            a = re.search(r'line (\d+)', ln)
            if "//## File" in ln and a:
                cur = (os.path.basename(re.search(r'File "([^"]+)"', ln).group(1)), int(a.group(1)))
                continue
            b = re.match(r'\s+/\*([0-9a-f]+)\*/', ln)
            if b and cur:
                m[int(b.group(1), 16)] = cur
        return m
    return {}


def main(rep, kregex, mangled, top=30):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kregex}"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    hdr = r[1]
    rows = r[2:]
    ai, ei, si = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[0][ai], 16)
    lm = line_map(mangled)
    agg = {}
    tot_e = tot_s = 0
    for x in rows:
        if len(x) <= max(ai, ei, si) or not x[ai].startswith("0x"):
            break                                   # next kernel's section
        off = int(x[ai], 16) - base
        e = int(x[ei]) if x[ei].isdigit() else 0
        s = int(x[si]) if x[si].isdigit() else 0
        tot_e += e
        tot_s += s
        k = lm.get(off, ("?", 0))
        a = agg.setdefault(k, [0, 0])
        a[0] += e
        a[1] += s
    print(f"total warp-instructions {tot_e:.3e}, samples {tot_s}")
    srcs = {}
    for (f, l), (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(top)]:
        if f not in srcs:
            p = os.path.join(ROOT, "paper_2605_20497_b200", "csrc", f)
            srcs[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = srcs[f][l - 1].strip() if 0 < l <= len(srcs[f]) else ""
        print(f"{100 * s / tot_s:5.1f}% smp {100 * e / tot_e:5.1f}% inst  {f}:{l}  {text[:80]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
