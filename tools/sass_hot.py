"""Hot SASS regions of one kernel from `ncu -i REP --page source --csv --print-source sass -k regex:K`
(run here): instructions executed per address, printed in address order for the top windows,
plus totals per opcode.  Usage: sass_hot.py CSV [min_share]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, ith, isa = (hdr.index(x) for x in ("Address", "Source", "Instructions Executed",
                                                   "Thread Instructions Executed", "# Samples"))
ins = []
for r in rows[2:]:
    try:
        ins.append((r[ia], r[isrc].strip(), int(r[iex]), int(r[ith]), int(r[isa])))
    except (ValueError, IndexError):
        pass
tot = sum(x[2] for x in ins) or 1
tots = sum(x[4] for x in ins) or 1
print("total warp instructions %.3e, samples %d" % (tot, tots))
op = Counter()
for a, s, e, t, sa in ins:
    o = s.split()[0] if s else "?"
    if o.startswith("@"):
        o = s.split()[1]
    op[o.split(".")[0]] += e
print("by opcode:", ", ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in op.most_common(25)))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
print("%-6s %6s %6s %5s  %s" % ("idx", "inst%", "samp%", "thr", "sass"))
for i, (a, s, e, t, sa) in enumerate(ins):
    if e / tot >= thr or sa / tots >= 0.01:
        print("%-6d %6.2f %6.2f %5.1f  %s" % (i, 100 * e / tot, 100 * sa / tots, t / e if e else 0, s[:110]))
