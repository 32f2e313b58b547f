"""Per-CUDA-source-line hot spots of one kernel launch in an .ncu-rep (read here, no GPU).
Usage: python tools/ncu_lines2.py REP KERNEL_FUNCTION_NAME [launch_skip] [top]"""
import csv, io, os, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      kname, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = os.path.basename(row[1]); continue
    if row[0] == "Function Name":
        func = row[1]; continue
    if row[0] == "Line No":
        hdr = row; continue
    if hdr is None or not row[0]:
        continue
    d = dict(zip(hdr[2:], row[2:]))
    try:
        rows.append((int(d.get("Warp Stall Sampling (All Samples)") or 0), int(d.get("Instructions Executed") or 0),
                     f"{fname}:{row[0]}", row[1].strip()[:100]))
    except ValueError:
        pass
tw = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"{func}\ntotal stall samples {tw}, warp-instructions {ti:.4e}")
for w, i, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*w/tw:5.1f}% stall {100*i/ti:5.1f}% inst  {ln:>18} {src}")
