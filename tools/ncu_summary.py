"""Summarise an ncu report: key metrics per kernel (reads `ncu -i --page details --csv`)."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Registers Per Thread', 'Executed Ipc Active',
        'Issue Slots Busy', 'Theoretical Occupancy', 'Block Limit Shared Mem', 'Dynamic Shared Memory Per Block',
        'Static Shared Memory Per Block']


def details(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    res = {}
    for r in rows[1:]:
        d = res.setdefault((r[ii], r[ki]), {})
        d.setdefault(r[mi], (r[vi], r[ui]))
    return res


def raw(rep, metrics):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        res.append({m: r[h.index(m)] for m in metrics if m in h} | {'Kernel Name': r[h.index('Kernel Name')]})
    return res


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        for (i, k), d in details(rep).items():
            print('==', i, k[:90])
            for m in WANT:
                if m in d:
                    print('   %-34s %s %s' % (m, d[m][0], d[m][1]))
        for r in raw(rep, ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum']):
            print('   raw', r)
