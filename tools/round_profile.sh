#!/bin/bash
# One GPU call's worth of round evidence -> gpurun_out/prof_<tag>/ : bench lines for
# every BASELINE workload (film512 f32 and f64 with the full-grid CPU reference legs),
# the reference arm (f32, f64), the GPU test log and smoke().
T=${1:-cur}; O=gpurun_out/prof_$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
(nproc; free -g) > $O/host.txt
python bench.py > $O/bench_film512.json 2> $O/bench_film512.err
python bench.py --precision 64 > $O/bench_film512_f64.json 2> $O/bench_film512_f64.err
for w in sp4 sp4fine cube128 film1024; do
  python bench.py --workload $w --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --workload cube128 --precision 64 --skip-cpu > $O/bench_cube128_f64.json 2> $O/bench_cube128_f64.err
python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --impl reference --steps 5 --warmup 2 --precision 64 > $O/bench_reference_f64.json 2> $O/bench_reference_f64.err
[ -z "$SKIP_TESTS" ] && python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
[ -z "$SKIP_TESTS" ] && python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
ls -la $O
