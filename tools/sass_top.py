"""Top SASS lines by stall samples from an ncu source page (csv.gz), with the
dominant stall reasons and the executed count:  python tools/sass_top.py src.csv.gz [n]"""
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
h = rows[hi]
S, A, SM, IE = h.index("Source"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
body = [r for r in rows[hi + 1:] if len(r) > SM and r[SM] not in ("", "Warp Stall Sampling (All Samples)")]
tot = sum(float(r[SM]) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for idx, r in sorted(enumerate(body), key=lambda x: -float(x[1][SM]))[:n]:
    rs = sorted(((float(r[i] or 0), h[i][6:]) for i in reasons), reverse=True)[:3]
    print(f"{idx:5d} {float(r[SM]) / tot:6.2%} {int(float(r[IE] or 0)):>10} {r[S].strip()[:58]:58s} " + " ".join(f"{b}:{a:.0f}" for a, b in rs))
