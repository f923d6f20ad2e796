"""Split a kernel's SASS (ncu source page) into regions between BAR.SYNC and
report instructions executed and stall samples per region + top opcodes."""
import csv
import re
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if 'Address' in r][0]
hdr = rows[hi]
S, IE, SM = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
regions, cur, ops = [], [0, 0, Counter(), Counter()], None
tot_i = tot_s = 0
for r in rows[hi + 1:]:
    if len(r) <= IE or r[IE] == 'Instructions Executed':
        continue
    src = r[S]
    ie = float(r[IE] or 0)
    sm = float(r[SM] or 0)
    tot_i += ie
    tot_s += sm
    op = src.split()[0] if src else ''
    if op.startswith('@'):
        op = src.split()[1]
    cur[0] += ie
    cur[1] += sm
    cur[2][op.split('.')[0]] += ie
    cur[3][op.split('.')[0]] += sm
    if 'BAR.SYNC' in src or 'EXIT' in src and ie > 0 and False:
        regions.append(cur)
        cur = [0, 0, Counter(), Counter()]
regions.append(cur)
print(f'total warp-instr {tot_i:.3e}, stall samples {tot_s:.0f}')
for n, (i, s, c, cs) in enumerate(regions):
    print(f'region {n}: instr {i / tot_i:6.1%}  samples {s / max(tot_s, 1):6.1%}  top: ' +
          ', '.join(f'{k}:{v / max(i, 1):.0%}' for k, v in c.most_common(8)))
