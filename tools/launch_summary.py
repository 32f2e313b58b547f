"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per-kernel launches, time, share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
            continue
        name = r[ki].split('(')[0].replace('void ', '').strip()
        v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f'# {sum(v[0] for v in agg.values())} launches, {tot:.3f} ms total (cold-cache, serialised: compare shares)')
    print(f'{"kernel":55s} {"launches":>8s} {"ms":>10s} {"share":>6s}')
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f'{k:55s} {c:8d} {ms:10.3f} {100 * ms / tot:5.1f}%')


if __name__ == '__main__':
    main(sys.argv[1])
