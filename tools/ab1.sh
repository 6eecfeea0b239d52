export PYTHONUNBUFFERED=1
out=gpurun_out/ab1; mkdir -p $out
QFT_LIB=$(realpath variants/g3.so) timeout 300 python tools/vcheck.py 4096 5 > $out/vcheck_g3.log 2>&1
QFT_LIB=$(realpath variants/g3s.so) timeout 300 python tools/vcheck.py 4096 5 > $out/vcheck_g3s.log 2>&1
bash tools/ab.sh -c 2 -r 3 paper_1301_0763_b200/libqftb200.so variants/g3.so variants/g3s.so > $out/ab_c2.log 2>&1
bash tools/ab.sh -c 4 -r 1 paper_1301_0763_b200/libqftb200.so variants/l2_40.so variants/l2_72.so variants/l2_104.so > $out/ab_c4.log 2>&1
bash tools/ab.sh -c 3 -r 1 paper_1301_0763_b200/libqftb200.so variants/l2_40.so variants/l2_72.so variants/l2_104.so > $out/ab_c3.log 2>&1
