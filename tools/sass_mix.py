"""Static SASS opcode mix of the kernels in an object: python tools/sass_mix.py obj regex"""
import collections
import re
import subprocess
import sys

txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r'\n\s+Function : ', txt)[1:]:
    name = f.split('\n')[0]
    if not re.search(sys.argv[2], name):
        continue
    ops = collections.Counter()
    for m in re.finditer(r'/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', f):
        ops[m.group(1).split('.')[0]] += 1
    fp = sum(ops[k] for k in ('FADD', 'FFMA', 'FMUL', 'DADD', 'DFMA', 'DMUL'))
    print(f"{name[:100]}\n   total {sum(ops.values())} fp {fp}  {ops.most_common(12)}")
