"""Print key `ncu --page details` metrics per kernel of an .ncu-rep (run here, no GPU)."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Executed Ipc Active', 'Issue Slots Busy', 'Block Limit Shared Mem', 'Block Limit Registers',
        'Dynamic Shared Memory Per Block', 'Static Shared Memory Per Block', 'Mem Busy', 'Max Bandwidth',
        'L2 Compression Success Rate']

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
res = {}
for r in rows[1:]:
    d = res.setdefault((int(r[ii]), r[ki].split('(')[0]), {})
    d.setdefault(r[mi], (r[vi], r[ui]))
for (i, k), d in sorted(res.items()):
    print('== %d %s' % (i, k))
    print('   ' + ' | '.join('%s=%s%s' % (w, d[w][0], d[w][1]) for w in WANT if w in d))
