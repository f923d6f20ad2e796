#!/bin/bash
# ncu evidence of the default bench command -> gpurun_out/<tag>/ :
# launch list (per-launch gpu__time_duration, clocks not locked) and one
# --set full capture (with source) of the five step kernels as an .ncu-rep.
T=${1:-cur}; O=gpurun_out/$T; mkdir -p $O
ARGS=${BENCH_ARGS:-}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu $ARGS > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches.csv $O/launches_summary.txt "ncu launch list of: python bench.py --steps 2 --warmup 3 --skip-cpu $ARGS" 2>&1 | tail -2
K="regex:k_r2c_x|k_fft_y_fwd|k_fft_z_conv|k_fft_y_inv|k_c2r_x_llg_v"
ncu --set full --import-source on --clock-control none -k "$K" --launch-skip ${SKIP:-10} -c 5 -o $O/full \
    python bench.py --steps 2 --warmup 3 --skip-cpu $ARGS > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/full.ncu-rep > $O/ncu_full_summary.txt 2>&1

# the .ncu-rep with source exceeds the 64 MiB pull limit: export the pages here
for k in k_r2c_x k_fft_y_fwd k_fft_z_conv k_fft_y_inv k_c2r_x_llg_v; do
  ncu -i $O/full.ncu-rep --page source --csv --kernel-name regex:$k --print-source sass 2>/dev/null | gzip > $O/src_$k.csv.gz
  ncu -i $O/full.ncu-rep --page source --csv --kernel-name regex:$k --print-source cuda 2>/dev/null | gzip > $O/srccu_$k.csv.gz
done
ncu -i $O/full.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/raw.csv.gz
[ -z "$KEEP_REP" ] && rm -f $O/full.ncu-rep

ls -la $O
