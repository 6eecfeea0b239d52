export PYTHONUNBUFFERED=1
out=gpurun_out/ab7; mkdir -p $out
QFT_LIB=$(realpath variants/split8.so) timeout 300 python tools/vcheck.py 4096 3 > $out/vcheck.log 2>&1
bash tools/ab.sh -c 2 -r 2 paper_1301_0763_b200/libqftb200.so variants/split2.so variants/split4.so variants/split8.so variants/split4e.so > $out/ab.log 2>&1
