"""Record one kernel of an ncu --set full capture into profiles/ncu_traffic.json (read by bench.py:
roofline.traffic / ncu, issue_roofline). usage: python tools/ncu_record.py REP KERNEL_REGEX WORKLOAD NAME SOURCE"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = {"dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
     "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
     "l2_hit_pct": "lts__t_sector_hit_rate.pct", "warp_instructions": "smsp__inst_executed.sum",
     "ipc_active": "sm__inst_executed.avg.per_cycle_active", "duration_ns": "gpu__time_duration.sum",
     "l1_data_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"}


def main(rep, kre, workload, name, source):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, val = rows[0], rows[1], rows[2]
    rec = {}
    for k, m in M.items():
        if m not in hdr:
            continue
        i = hdr.index(m)
        x = float(val[i].replace(",", ""))
        u = units[i]
        if "bytes" in k:
            x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        if k == "duration_ns":
            x *= {"ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(u, 1)
        rec[k] = x
    rec["dram_bytes_per_launch"] = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
    rec["duration_ms"] = rec.pop("duration_ns", 0) / 1e6
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d.setdefault("_doc", "per-launch counters of the named kernels from ncu --set full --clock-control none "
                 "captures (tools/ncu_record.py); read by bench.py (roofline.traffic / ncu, issue_roofline)")
    rec["source"] = source
    d.setdefault(workload, {})[name] = rec
    json.dump(d, open(p, "w"), indent=1)
    print(name, json.dumps(rec))


if __name__ == "__main__":
    main(*sys.argv[1:])
