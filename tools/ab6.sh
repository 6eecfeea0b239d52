export PYTHONUNBUFFERED=1
out=gpurun_out/ab6; mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
bash tools/ab.sh -c 2 -r 3 variants/sc.so paper_1301_0763_b200/libqftb200.so > $out/ab_c2.log 2>&1
bash tools/ab.sh -c 5 -r 1 variants/sc.so paper_1301_0763_b200/libqftb200.so > $out/ab_c5.log 2>&1
bash tools/ab.sh -c 3 -r 1 variants/sc.so paper_1301_0763_b200/libqftb200.so > $out/ab_c3.log 2>&1
