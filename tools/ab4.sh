export PYTHONUNBUFFERED=1
out=gpurun_out/ab4; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
bash tools/ab.sh -c 2 -r 3 variants/sc.so paper_1301_0763_b200/libqftb200.so > $out/ab_c2.log 2>&1
bash tools/ab.sh -c 5 -r 1 variants/sc.so paper_1301_0763_b200/libqftb200.so > $out/ab_c5.log 2>&1
bash tools/ab.sh -c 3 -r 1 variants/sc.so paper_1301_0763_b200/libqftb200.so > $out/ab_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qft_cdft_pipe" -s 3 -c 1 -o $out/prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $out/ncu2.log 2>&1
