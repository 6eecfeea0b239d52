#!/bin/bash
# Round-2 GPU cycle: gpu tests, bench lines for every config, launch lists.
# usage (inside gpurun): bash tools/r2_cycle.sh <tag>
export PYTHONUNBUFFERED=1
tag=${1:-r2}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt 2>&1
lscpu | head -20 >> $out/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> $out/pytest_gpu.log
timeout 400 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
for c in 1 3 4 5; do timeout 500 python bench.py --config $c > $out/bench_c$c.json 2> $out/bench_c$c.err; done
timeout 400 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err
for c in 2 3 4 5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"qft_|lg_" -c 40 --csv --log-file $out/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
done
echo done > $out/status
