#!/bin/bash
# Round-end measurement on one B200 (inside gpurun): bench lines for every
# config, the reference arm, launch lists and ncu full captures of the top kernels,
# summarised on the box (the .ncu-rep files of the multi-pass items are large).
# usage: bash tools/final_measure.sh [tag]   (outputs under gpurun_out/<tag>/)
export PYTHONUNBUFFERED=1
tag=${1:-final}
out=gpurun_out/$tag; mkdir -p $out
timeout 400 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
for c in 1 3 4 5; do timeout 500 python bench.py --config $c > $out/bench_c$c.json 2> $out/bench_c$c.err; done
timeout 400 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err
for c in 2 3 4 5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"qft_|lg_" -c 40 --csv --log-file $out/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"qft_cdft_(smem|pipe)" -s 3 -c 1 -o $out/prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qft_cdft_smem -s 1 -c 1 -o $out/prof_c5 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lg_item -s 1 -c 1 -o $out/prof_c3 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lg_item -s 1 -c 1 -o $out/prof_c4 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python tools/make_summary.py $out $out/summary.json $tag > /dev/null 2>&1
for c in 2 3 4 5; do
  case $c in 2) b=16384;; 3) b=2048;; 4) b=64;; *) b=262144;; esac
  python tools/prof_summary.py $out/prof_c$c.ncu-rep $b > $out/prof_c$c.txt 2>&1
  python tools/prof_stalls.py $out/prof_c$c.ncu-rep >> $out/prof_c$c.txt 2>&1
done
rm -f $out/prof_c3.ncu-rep $out/prof_c4.ncu-rep
timeout 300 python tools/size_sweep.py --json $out/size_sweep.json > $out/size_sweep.txt 2>&1
timeout 300 python tools/size_sweep.py --algo classical --json $out/size_sweep_classical.json > $out/size_sweep_classical.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"cl_" -c 60 --csv --log-file $out/launches_classical_c4.csv python tools/classical_prof.py 20 64 f64 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cl_tree -s 2 -c 1 -o $out/prof_classical_c2 python tools/classical_prof.py 12 16384 > /dev/null 2>&1
python tools/prof_summary.py $out/prof_classical_c2.ncu-rep 16384 > $out/prof_classical_c2.txt 2>&1
python tools/prof_stalls.py $out/prof_classical_c2.ncu-rep >> $out/prof_classical_c2.txt 2>&1
rm -f $out/prof_classical_c2.ncu-rep $out/prof_c2.ncu-rep $out/prof_c5.ncu-rep
echo done > $out/status
