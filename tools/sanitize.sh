#!/bin/bash
# compute-sanitizer runs over the GPU kernels -> gpurun_out/<tag>/san_*.log
#   memcheck  : out-of-bounds / misaligned accesses (every step kernel incl. TMA, cp.async paths)
#   racecheck : shared-memory hazards (FFT stage barriers, K5 block_finish, K3 in-place cp.async)
#   synccheck : illegal barrier use
# on tests that cover K5's last-block sample combine, relax's device skip flags,
# the fused K1-in-K5 chunks and the production (C2/C3-class) variants, plus a
# short C4 bench (memcheck only; racecheck of 5x16M-cell passes is too slow).
T=${1:-san}; O=gpurun_out/$T; mkdir -p $O
CS=compute-sanitizer
SEL="test_sample_and_energies or test_relax_stops_at_reference_step or test_relax_exhausts or test_steps_with_demag or test_nonfinite or test_step_async_error"
run() { local name=$1; shift; echo "== $*" > $O/san_$name.log; timeout ${TO:-900} "$@" >> $O/san_$name.log 2>&1; echo "rc=$?" >> $O/san_$name.log; tail -4 $O/san_$name.log; }
run memcheck_parity  $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL"
run memcheck_fusion  $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_fusion.py -q -x
run memcheck_prod    $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_production.py -q -x -k "c2 or 128x128x64_f32"
run racecheck_parity $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL"
run racecheck_fusion $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest tests/test_gpu_fusion.py -q -x -k "32-16-4 or 128-32-1"
run synccheck_parity $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL"
TO=1200 run memcheck_bench_c4 $CS --tool memcheck --error-exitcode 9 python bench.py --steps 3 --warmup 3 --skip-cpu
TO=1200 run racecheck_bench_sp4fine $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python bench.py --workload sp4fine --steps 2 --warmup 3 --skip-cpu
TO=1200 run racecheck_bench_cube $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python bench.py --workload cube128 --steps 1 --warmup 3 --skip-cpu
ls -la $O
