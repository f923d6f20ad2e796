#!/bin/bash
# SASS proof of the Blackwell features in the production kernels (no GPU needed):
# TMA loads (UTMALDG), mbarrier sync (SYNCS.*), L2 bulk prefetch (UBLKPF) and cp.async
# (LDGSTS) per kernel, with the instruction lines.  -> profiles/<tag>/sass_evidence.txt
T=${1:-r2}; O=profiles/$T; mkdir -p $O
OBJ=paper_1406_7459_b200/build/engine_f32.o
cuobjdump -sass $OBJ > /tmp/sass_f32.txt
python3 - /tmp/sass_f32.txt > $O/sass_evidence.txt <<'PY'
import re, subprocess, sys
txt = open(sys.argv[1]).read().split("Function : ")
want = ["k_fft_y_fwd_tmaIfLi1024ELb1", "k_fft_y_inv_tmaIfLi1024ELb1", "k_fft_z_conv2IfLi128ELb1ELb1",
        "k_r2c_xIfLi512ELi0ELb0", "k_c2r_x_llg_vIfLi512ELb0ELi0ELb0ELb0"]
pat = re.compile(r"\b(UTMALDG|UTMASTG|UBLKCP|UBLKPF|SYNCS\.[A-Z.0-9]+|LDGSTS\.[A-Z.0-9]+|UTMAPF|FENCE\.VIEW\.ASYNC\.S)\b")
print("# cuobjdump -sass paper_1406_7459_b200/build/engine_f32.o (sm_100a): Blackwell async-copy / barrier")
print("# instructions in the C4 f32 production kernels (tools/sass_evidence.sh)\n")
for blk in txt[1:]:
    name = blk.split("\n", 1)[0].strip()
    if not any(w in name for w in want):
        continue
    dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    hits = [l.strip() for l in blk.split("\n") if pat.search(l)]
    counts = {}
    for l in hits:
        k = pat.search(l).group(1)
        counts[k] = counts.get(k, 0) + 1
    print(f"== {dn}\n   counts: {counts}")
    seen = set()
    for l in hits:
        k = pat.search(l).group(1)
        if k in seen:
            continue
        seen.add(k)
        print("   " + re.sub(r"\s+", " ", l)[:150])
    print()
PY
cat $O/sass_evidence.txt
