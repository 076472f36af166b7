"""Summarise an ncu launch list (gpu__time_duration, optional dram bytes) per kernel."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
d = defaultdict(lambda: defaultdict(list))
order = []
for r in rows[1:]:
    k = r[ki][:80]
    if k not in d:
        order.append(k)
    d[k][r[mi]].append(float(r[vi].replace(',', '')))
for k in order:
    v = d[k]
    t = sum(v['gpu__time_duration.sum']) / len(v['gpu__time_duration.sum']) / 1000
    b = sum(v['dram__bytes_read.sum']) / len(v['dram__bytes_read.sum']) / 1e6 if v['dram__bytes_read.sum'] else 0
    print('%4d x %7.1f us %7.1f MB %6.0f GB/s  %s' % (len(v['gpu__time_duration.sum']), t, b, b / t * 1e3 if t else 0, k))
