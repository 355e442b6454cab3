#!/usr/bin/env python
"""Aggregate an ncu launch-list CSV (gpu__time_duration + dram bytes) per kernel.

    python tools/launch_table.py gpurun_out/launches_target.csv [--steps 2]
"""
import collections
import csv
import io
import sys

UNIT = {'ms': 1e-3, 'us': 1e-6, 'ns': 1e-9, 'msecond': 1e-3, 'usecond': 1e-6, 'nsecond': 1e-9,
        'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}


def table(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
    agg = collections.defaultdict(lambda: [set(), 0.0, 0.0])
    for r in rows:
        n = r['Kernel Name']
        short = 'cutlass_int8_gemm' if 'cutlass' in n else n.split('(')[0].replace('void ', '').replace('tci::<unnamed>::', '')[:48]
        v = float(r['Metric Value'].replace(',', '')) * UNIT.get(r['Metric Unit'], 1)
        a = agg[short]
        a[0].add(r['ID'])
        if r['Metric Name'] == 'gpu__time_duration.sum':
            a[1] += v
        else:
            a[2] += v
    return agg


if __name__ == '__main__':
    steps = int(sys.argv[sys.argv.index('--steps') + 1]) if '--steps' in sys.argv else 1
    agg = table(sys.argv[1])
    tot = sum(a[1] for k, a in agg.items() if not k.startswith('at::') and 'elementwise' not in k)
    for k, a in sorted(agg.items(), key=lambda t: -t[1][1]):
        if a[1] < 1e-5:
            continue
        print(f"{k:50s} n/step={len(a[0]) / steps:5.1f} {a[1] * 1e3 / steps:8.2f} ms/step "
              f"{100 * a[1] / tot:5.1f}% {a[2] / 1e9 / steps:7.2f} GB/step {a[2] / a[1] / 1e12 if a[1] else 0:5.2f} TB/s")
    print(f"own kernels total {tot * 1e3 / steps:.2f} ms/step")
