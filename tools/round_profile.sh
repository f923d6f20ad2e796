#!/bin/bash
# One GPU call's worth of round evidence -> gpurun_out/prof_<tag>/ :
# bench lines for every BASELINE workload (+ fp64, + the reference arm), the
# ncu launch list of the default bench command and one ncu --set full capture
# of the step kernels (summaries only; the .ncu-rep stays on the box).
T=${1:-cur}; O=gpurun_out/prof_$T; mkdir -p $O
python bench.py > $O/bench_film512.json 2> $O/bench_film512.err
python bench.py --precision 64 --skip-cpu > $O/bench_film512_f64.json 2> $O/bench_film512_f64.err
for w in sp4 sp4fine cube128 film1024; do
  python bench.py --workload $w --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches.csv $O/launches_summary.txt "ncu launch list of: python bench.py --steps 2 --warmup 3 --skip-cpu" 2>&1 | tail -2
K="regex:k_r2c_x|k_fft_y_fwd|k_fft_z_conv|k_fft_y_inv|k_c2r_x_llg_v"
ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 10 -c 5 -o /tmp/full_$T \
    python bench.py --steps 2 --warmup 3 --skip-cpu > $O/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/full_$T.ncu-rep > $O/ncu_full_summary.txt
ncu -i /tmp/full_$T.ncu-rep --page raw --csv > $O/ncu_full_raw.csv
for k in k_r2c_x k_fft_y_fwd k_fft_z_conv k_fft_y_inv k_c2r_x_llg_v; do
  echo "== $k" >> $O/stall_lines.txt
  python tools/stall_lines.py /tmp/full_$T.ncu-rep $k 12 >> $O/stall_lines.txt 2>&1
done
ls -la $O
