"""One-screen summary of a bench.py JSON line (for tools/gpu.sh)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    print(path, "ms/step %.3f" % d["ms_per_step"], "pins/s %.3e" % d["value"], "V", d["config"].get("V"))
    print("  step_ms", d.get("step_ms"))
    print("  kernels", list(d.get("kernels_ms", {}).items())[:8])
    r = d.get("roofline") or {}
    print("  roofline", r.get("kernel"), "frac %.4f" % r.get("frac", 0), "ms/launch", r.get("ms_per_launch"))
    h = d.get("hierarchy")
    if h:
        print("  hierarchy ms %.1f levels %d" % (h["total_coarsening_ms"], h["levels"]), h.get("level_ms", [])[:6],
              h.get("phase_ms_total", ""))
    if d.get("e2e"):
        print("  e2e %.3e" % d["e2e"]["value"])
    print("  clocks", d.get("clocks"))
