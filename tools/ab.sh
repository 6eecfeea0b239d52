#!/bin/bash
# A/B timing of library variants (inside gpurun): bash tools/ab.sh [-c CONFIG] lib1.so lib2.so ...
export PYTHONUNBUFFERED=1
cfg=2
if [ "$1" = "-c" ]; then cfg=$2; shift 2; fi
for lib in "$@"; do
  v=$(QFT_LIB=$(realpath $lib) timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(f\"{l['value']/1e6:.3f}M tr/s frac {l['roofline']['frac']:.3f} parity {l['parity_bitwise_sampled']}\")" 2>&1)
  echo "config $cfg $lib: $v"
done
