#!/bin/bash
# build (here) + run (on the GPU box) the phase probe: tools/probe/run_probe.sh build|run [LOG2N] [extra nvcc -D...]
cd "$(dirname "$0")"
if [ "$1" = build ]; then
  l=${2:-12}; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr \
    -DPLOG2N=$l "$@" phase_probe.cu -o probe_$l
else
  for f in probe_*; do echo "== $f"; ./$f; done
fi
