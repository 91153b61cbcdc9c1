"""Per CUDA source line: warp-stall samples and warp instructions executed, from an .ncu-rep
(`ncu -i REP --page source --print-source cuda,sass --csv -k regex:KERNEL`).  Run here."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k',
                      'regex:' + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, agg, hdr = None, {}, None
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == '' or r[0] == '-':
        continue
    try:
        s, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    agg[(fname, int(r[0]))] = (s, ins, r[1][:90])
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print('total samples %d, warp instructions %.3e' % (tot_s, tot_i))
key = 1 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 0
for (f, ln), (s, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print('%5.1f%% samp %5.1f%% inst  %s:%d  %s' % (100 * s / tot_s, 100 * ins / tot_i, f, ln, src))
