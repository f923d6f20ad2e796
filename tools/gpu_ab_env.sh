#!/bin/bash
# A/B of library variants and env switches: tools/gpu_ab_env.sh tag "label:ENV=.. MFD_LIB=variants/x.so" ...
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for rep in 1 2; do
  for spec in "$@"; do
    lab=${spec%%:*}; env=${spec#*:}
    env $env python bench.py --skip-cpu --steps 300 --warmup 10 ${BENCH_ARGS:-} > $O/ab_${lab}_$rep.json 2> $O/ab_${lab}_$rep.err
    python - $O/ab_${lab}_$rep.json $lab <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    print(f"{sys.argv[2]:14s} ms={d['ms_per_step']:.4f} frac={d['step_roofline']['frac']:.3f}", {k: round(v,4) for k,v in d['per_kernel_ms'].items()})
except Exception as e: print(sys.argv[2], 'fail', e)
PY
  done
done | tee $O/ab_summary.txt
