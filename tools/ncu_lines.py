"""Aggregate ncu source-page (cuda,sass) metrics per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > f.csv; python ncu_lines.py f.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == 'Line No'][0]
i_line, i_src = 0, 1
i_samp = hdr.index('Warp Stall Sampling (All Samples)')
i_exec = hdr.index('Instructions Executed')
agg = {}
cur = None
src = {}
for r in rows:
    if not r or r[0] in ('Line No', 'File Path', 'Function Name'):
        continue
    if r[0].strip().isdigit():
        cur = int(r[0])
        src[cur] = r[1]
    if len(r) > i_exec and r[i_exec].strip().isdigit() and cur is not None:
        a = agg.setdefault(cur, [0, 0])
        a[0] += int(r[i_exec])
        a[1] += int(r[i_samp]) if r[i_samp].strip().isdigit() else 0
te = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for ln, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print('%5d inst %5.1f%% stall %5.1f%%  %s' % (ln, 100 * e / te, 100 * s / ts, src.get(ln, '')[:90]))
