"""Instruction-class histogram of an ncu SASS source page (csv.gz from
tools/ncu_round.sh), weighted by 'Instructions Executed' (warp level), with
stall samples: python tools/sass_hist.py src_<kernel>.csv.gz [top]"""
import csv
import gzip
import re
import sys
from collections import defaultdict

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
h = rows[hi]
S, IE, SM = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hi + 1:] if len(r) > IE and r[IE] not in ("", "Instructions Executed")]
cls = defaultdict(lambda: [0, 0.0])
tot_i = tot_s = 0
for r in body:
    src = r[S].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    op = m.group(2) if m else src.split()[0]
    mod = (m.group(3) or "") if m else ""
    key = op + (mod if op in ("LDG", "STG", "LDS", "STS", "LDL", "STL", "LDGSTS", "SHFL", "MUFU") else "")
    n = int(float(r[IE] or 0))
    s = float(r[SM] or 0)
    cls[key][0] += n
    cls[key][1] += s
    tot_i += n
    tot_s += s
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,.0f}")
for k, (n, s) in sorted(cls.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{k:22s} {n:14,d} {n / tot_i:6.1%}  stalls {s / max(tot_s, 1):6.1%}")
