#!/bin/bash
# ncu --set full of one kernel (regex $2) of a bench command; exports the SASS source page.
# tools/ncu_one.sh <tag> <kernel-regex> <bench args...>
T=$1; K=$2; shift 2; O=gpurun_out/$T; mkdir -p $O
ncu --set full --import-source on --clock-control none -k "regex:$K" --launch-skip ${SKIP:-2} -c 1 -o $O/one \
    python bench.py --steps 2 --warmup 3 --skip-cpu "$@" > $O/ncu_one.log 2>&1
python tools/ncu_summary.py $O/one.ncu-rep > $O/ncu_one_summary.txt 2>&1
ncu -i $O/one.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/src_one.csv.gz
ncu -i $O/one.ncu-rep --page details --csv 2>/dev/null | gzip > $O/details_one.csv.gz
rm -f $O/one.ncu-rep
