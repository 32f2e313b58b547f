"""Instruction / stall-sample share per line range of a kernel (phases), from an .ncu-rep.
usage: python tools/ncu_phases.py REP KERNEL_REGEX MANGLED FILE name:a-b [name:a-b ...]"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit('/', 1)[0])
import ncu_lines  # noqa: E402


def main(rep, kre, mangled, fname, *ranges):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    hdr, rows = r[1], r[2:]
    ai, ei, si = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[0][ai], 16)
    lm = ncu_lines.line_map(mangled)
    ph = [(x.split(':')[0], *map(int, x.split(':')[1].split('-'))) for x in ranges]
    acc = {p[0]: [0, 0] for p in ph}
    acc['other'] = [0, 0]
    te = ts = 0
    for x in rows:
        if len(x) <= max(ai, ei, si) or not x[ai].startswith("0x"):
            break                                   # next kernel's section
        e = int(x[ei]) if x[ei].isdigit() else 0
        s = int(x[si]) if x[si].isdigit() else 0
        te += e
        ts += s
        f, l = lm.get(int(x[ai], 16) - base, ("?", 0))
        key = 'other'
        if f == fname:
            for name, a, b in ph:
                if a <= l <= b:
                    key = name
        acc[key][0] += e
        acc[key][1] += s
    print(f"total {te:.3e} warp-instructions")
    for k, (e, s) in acc.items():
        print(f"{k:20s} inst {100 * e / te:5.1f}%  samples {100 * s / ts:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
