export PYTHONUNBUFFERED=1
out=gpurun_out/ab5; mkdir -p $out
QFT_LIB=$(realpath variants/g3.so) timeout 300 python tools/vcheck.py 4096 3 > $out/vcheck_g3.log 2>&1
bash tools/ab.sh -c 2 -r 2 paper_1301_0763_b200/libqftb200.so variants/g3.so variants/umap0.so variants/nwa4.so variants/nwa6.so > $out/ab_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qft_cdft_pipe" -s 3 -c 1 -o $out/prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $out/ncu2.log 2>&1
