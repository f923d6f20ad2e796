#!/bin/bash
# A/B of library variants on the default bench workload: tools/gpu_ab.sh tag lib1 lib2 ...
# ("default" = the in-tree library).  Interleaved, two rounds each.
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then L=""; else L="MFD_LIB=variants/$v.so"; fi
    env $L python bench.py --skip-cpu --steps 400 --warmup 10 ${BENCH_ARGS:-} > $O/ab_${v}_$rep.json 2> $O/ab_${v}_$rep.err
    python - $O/ab_${v}_$rep.json $v <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    print(f"{sys.argv[2]:12s} ms={d['ms_per_step']:.4f} frac={d['step_roofline']['frac']:.3f}", {k: round(v,4) for k,v in d['per_kernel_ms'].items()})
except Exception as e: print(sys.argv[2], 'fail', e)
PY
  done
done | tee $O/ab_summary.txt
