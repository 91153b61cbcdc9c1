"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per launch)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h = rows[hi]
ki, mi, vi, ii, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID'), h.index('Metric Unit')
k = OrderedDict()
for r in rows[hi + 1:]:
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    if u == 'ns': v /= 1e6
    elif u == 'us' or u == 'usecond': v /= 1e3
    elif u in ('byte',): v /= 1e9
    elif u == 'Kbyte': v /= 1e6
    elif u == 'Mbyte': v /= 1e3
    elif u == 'Gbyte': pass
    elif u == 'msecond' or u == 'ms': pass
    k.setdefault((int(r[ii]), r[ki].split('(')[0][-40:]), {})[r[mi]] = v
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
items = list(k.items())[skip:]
tot = sum(m.get('gpu__time_duration.sum', 0) for _, m in items)
print('total %.3f ms over %d launches' % (tot, len(items)))
agg = OrderedDict()
for (i, name), m in items:
    a = agg.setdefault(name, [0, 0, 0, 0])
    a[0] += m.get('gpu__time_duration.sum', 0); a[1] += m.get('dram__bytes_read.sum', 0); a[2] += m.get('dram__bytes_write.sum', 0); a[3] += 1
for name, (t, r, w, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print('%-42s n=%3d %8.3f ms (%4.1f%%)  R %7.3f GB  W %7.3f GB  %6.2f TB/s' % (name, n, t, 100 * t / tot, r, w, (r + w) / t if t else 0))
