export PYTHONUNBUFFERED=1
out=gpurun_out/ab13; mkdir -p $out
bash tools/ab.sh -c 4 -r 2 variants/nostg.so paper_1301_0763_b200/libqftb200.so variants/stg128.so > $out/ab_c4.log 2>&1
QFT_LIB=$(realpath variants/stg128.so) timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "20 or 17 or 16" > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
rm -f variants/*.so
