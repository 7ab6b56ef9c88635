"""Compare two ncu launch lists (csv, --metrics gpu__time_duration.sum,dram__bytes_*) launch by launch."""
import collections
import csv
import io
import sys


def load(f):
    lines = [l for l in open(f) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO(''.join(lines))))
    L = collections.OrderedDict()
    for r in rows:
        i = int(r['ID'])
        L.setdefault(i, {'name': r['Kernel Name'].split('(')[0].replace('sgf::', '').replace('void ', ''),
                         'grid': r['Grid Size']})
        L[i][r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
    return L


A, B = load(sys.argv[1]), load(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 100.0
ta = tb = 0
for i in A:
    a, b = A[i], B.get(i)
    if b is None:
        continue
    t1, t2 = a['gpu__time_duration.sum'] / 1e3, b['gpu__time_duration.sum'] / 1e3
    b1 = (a['dram__bytes_read.sum'] + a['dram__bytes_write.sum']) / 1e9
    b2 = (b['dram__bytes_read.sum'] + b['dram__bytes_write.sum']) / 1e9
    ta += t1
    tb += t2
    if t1 > thr:
        print(i, a['name'][:30], '|', b['name'][:30], f"{t1:7.1f} -> {t2:7.1f} us  {b1:.3f} -> {b2:.3f} GB  {b2 / t2 * 1e3:.2f} TB/s")
print(f"sum {ta:.1f} -> {tb:.1f} us")
