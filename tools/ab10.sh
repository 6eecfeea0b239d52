export PYTHONUNBUFFERED=1
out=gpurun_out/ab10; mkdir -p $out
timeout 300 python tools/vcheck.py 16384 2 > $out/vcheck.log 2>&1
timeout 300 python tools/vcheck.py 8192 2 >> $out/vcheck.log 2>&1
bash tools/ab.sh -c 5 -r 2 variants/nopre.so paper_1301_0763_b200/libqftb200.so variants/pre8.so variants/pre2.so > $out/ab.log 2>&1
