#!/bin/bash
# one GPU cycle: parity tests, bench, then ncu of the smem kernel (only if the plain run exited 0)
# usage (inside gpurun): bash tools/gpu_cycle.sh <tag> [extra bench args]
tag=${1:-x}; shift
export PYTHONUNBUFFERED=1
timeout 500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 "$@" > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
timeout 120 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qft_cdft_smem -s 3 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu.log
