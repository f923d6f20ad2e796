#!/bin/bash
# usage: ab.sh label "ENV=.. ENV2=.." [bench args]
j() { python - "$1" <<'PY'
import json,sys
for l in open(sys.argv[1]).read().splitlines():
    if l.startswith('{'):
        d=json.loads(l)
if 'd' in dir():
    print(f"ms={d['ms_per_step']:.4f} frac={d['step_roofline']['frac']:.3f} ", {k: round(v,4) for k,v in d['per_kernel_ms'].items()})
else: print('no json')
PY
}
for spec in "$@"; do
  lab=${spec%%:*}; env=${spec#*:}
  env $env python bench.py --skip-cpu --steps 300 --warmup 10 ${BENCH_ARGS:-} > gpurun_out/ab_$lab.json 2> gpurun_out/ab_$lab.err
  echo "$lab [$env]: $(j gpurun_out/ab_$lab.json) $(tail -1 gpurun_out/ab_$lab.err | cut -c1-200)"
done
