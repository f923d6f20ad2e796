"""Top SASS lines of a kernel by stall samples, with the dominant reasons:
python tools/stall_lines.py report.ncu-rep kernel_regex [n]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if 'Address' in r][0]
h = rows[hi]
S, A, SM = h.index('Source'), h.index('Address'), h.index('Warp Stall Sampling (All Samples)')
reasons = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
body = [r for r in rows[hi + 1:] if len(r) > SM and r[SM] not in ('', 'Warp Stall Sampling (All Samples)')]
tot = sum(float(r[SM]) for r in body)
reason_tot = {}
for r in body:
    for i in reasons:
        reason_tot[h[i]] = reason_tot.get(h[i], 0) + float(r[i] or 0)
print('kernel total samples', tot, ' reasons:',
      ', '.join(f'{k[6:]}={v / tot:.0%}' for k, v in sorted(reason_tot.items(), key=lambda x: -x[1])[:8]))
for idx, r in sorted(enumerate(body), key=lambda x: -float(x[1][SM]))[:n]:
    rs = sorted(((float(r[i] or 0), h[i][6:]) for i in reasons), reverse=True)[:3]
    print(f'{idx:5d} {r[A]:>6} {float(r[SM]) / tot:6.2%} {r[S][:60]:60s} ' + ' '.join(f'{b}:{a:.0f}' for a, b in rs))
