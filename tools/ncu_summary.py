"""Summarise an .ncu-rep (read here, no GPU): key metrics + top stall reasons per kernel."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Warp Cycles Per Issued Instruction', 'Issue Slots Busy',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Ipc Active', 'Avg. Active Threads Per Warp',
        'Block Limit Shared Mem', 'Block Limit Registers', 'Dynamic Shared Memory Per Block', 'Grid Size',
        'Block Size', 'Branch Efficiency']


def main(path, raw_extra=()):
    det = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    ki, ii, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'ID', 'Metric Name', 'Metric Value', 'Metric Unit'))
    cur = None
    for row in r[1:]:
        if row[mi] in WANT:
            if row[ii] != cur:
                cur = row[ii]
                print(f'--- [{cur}] {row[ki][:90]}')
            print(f'   {row[mi]:40s} {row[vi]} {row[ui]}')
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    for row in rr[2:]:
        name = row[hh.index('Kernel Name')][:70]
        st = []
        for i, col in enumerate(hh):
            if col.startswith('smsp__pcsamp_warps_issue_stalled_') and not col.endswith('not_issued'):
                try:
                    st.append((float(row[i].replace(',', '')), col.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        top = sorted(st, reverse=True)[:6]
        print(f'stalls {name}: ' + ', '.join(f'{n} {100 * v / tot:.0f}%' for v, n in top))
        for m in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
                  'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active') + tuple(raw_extra):
            if m in hh:
                print(f'   {m} = {row[hh.index(m)]}')


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2:])
