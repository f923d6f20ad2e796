"""Aggregate an ncu capture's per-instruction counts and stall samples by CUDA
source line (nvdisasm -g on the kernel's cubin maps SASS offsets to lines).
python tools/sass_lines.py report.ncu-rep object.o ncu_kernel_regex mangled_regex [n]"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern, mkern = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
n = int(sys.argv[5]) if len(sys.argv) > 5 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if 'Address' in r][0]
h = rows[hi]
A, IE, SM = h.index('Address'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
body = []
for r in rows[hi + 1:]:
    if len(r) <= SM or not re.fullmatch(r'0x[0-9a-fA-F]+', r[A]):
        if body:
            break   # first copy only
        continue
    body.append((int(r[A], 16), float(r[IE] or 0), float(r[SM] or 0)))
base = body[0][0]
# line info of the matching function in the cubin
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
func = None
line = None
off2line = {}
want = None
for l in dis.splitlines():
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m:
        func = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and func and re.search(mkern, func):
        if want is None:
            want = func
        if func == want:
            off2line[int(m.group(1), 16)] = line
ie_l, sm_l = collections.Counter(), collections.Counter()
for a, ie, sm in body:
    ln = off2line.get(a - base, '?')
    ie_l[ln] += ie
    sm_l[ln] += sm
ti, ts = sum(ie_l.values()), sum(sm_l.values())
print(f"function {want[:90]}\n instr {ti:.3e}  samples {ts:.0f}")
for ln, v in ie_l.most_common(n):
    print(f"{ln:28s} instr {v / ti:6.1%}  stall {sm_l[ln] / ts:6.1%}")
