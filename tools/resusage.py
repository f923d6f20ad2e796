import sys,re,subprocess
pat = sys.argv[2] if len(sys.argv) > 2 else ''
out = subprocess.run(['cuobjdump','--dump-resource-usage',sys.argv[1]],capture_output=True,text=True).stdout
lines = out.splitlines()
for a,b in zip(lines, lines[1:]):
    m = re.search(r'Function (\S+):', a); r = re.search(r'REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)', b)
    if not (m and r): continue
    name = subprocess.run(['c++filt', m.group(1)], capture_output=True, text=True).stdout.strip()
    name = re.sub(r'\(.*', '', name)
    if re.search(pat, name):
        print(f'{name:45s} reg={r.group(1):4s} stack={r.group(2):5s} local={r.group(4)}')
