"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
h = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
agg = defaultdict(list)
for r in data:
    agg[r[ki].split('(')[0]].append(float(r[vi].replace(',', '')) * scale[r[ui]])
step = {k: v for k, v in agg.items() if any(s in k for s in ('r2c', 'fft', 'c2r', 'local_llg', 'yz'))}
tot = sum(sum(v) / len(v) for v in step.values())
with open(dst, 'w') as f:
    f.write(f'# {sys.argv[3] if len(sys.argv) > 3 else src}\n')
    for k, v in agg.items():
        avg = sum(v) / len(v)
        tag = f'share_of_step={avg / tot:.3f}' if k in step else '(setup, once)'
        f.write(f'{k:45s} launches={len(v):3d} avg_ms={avg:.4f} {tag}\n')
    f.write(f'sum of per-step kernel averages: {tot:.4f} ms\n')
print(open(dst).read())
