export PYTHONUNBUFFERED=1
out=gpurun_out/prof2; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lg_item" -s 1 -c 1 -o $out/prof_c3 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $out/ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qft_cdft_smem" -s 1 -c 1 -o $out/prof_c5 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $out/ncu5.log 2>&1
