export PYTHONUNBUFFERED=1
out=gpurun_out/ab16; mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
bash tools/ab.sh -c 4 -r 2 variants/norot.so paper_1301_0763_b200/libqftb200.so > $out/ab_c4.log 2>&1
rm -f variants/*.so
