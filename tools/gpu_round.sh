#!/bin/bash
# One GPU call: GPU tests, smoke, default bench line (with the full-grid CPU
# baseline) and the reference arm -> gpurun_out/<tag>/
T=${1:-cur}; O=gpurun_out/$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=25 ${PYTEST_ARGS} > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/ref.json 2> $O/ref.err
ls -la $O
