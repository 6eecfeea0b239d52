#!/bin/bash
# A/B timing of library variants (inside gpurun): bash tools/ab.sh [-c CONFIG] [-r ROUNDS] lib1.so lib2.so ...
# Each round times every library once (interleaved, so box drift hits all variants alike).
export PYTHONUNBUFFERED=1
cfg=2; rounds=2
while [ "${1:0:1}" = "-" ]; do
  case $1 in -c) cfg=$2; shift 2;; -r) rounds=$2; shift 2;; *) shift;; esac
done
for r in $(seq $rounds); do
for lib in "$@"; do
  v=$(QFT_LIB=$(realpath $lib) timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); p=l['parity']; print(f\"{l['value']/1e6:.3f}M tr/s frac {l['roofline']['frac']:.3f} parity {p['mismatches']}/{p['rows_checked']}\")" 2>&1)
  echo "round $r config $cfg $lib: $v"
done
done
