export PYTHONUNBUFFERED=1
out=gpurun_out/r2v; mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
bash tools/ab.sh -c 4 -r 2 variants/nostg.so paper_1301_0763_b200/libqftb200.so > $out/ab_c4.log 2>&1
rm -f variants/nostg.so
grep -q "rc=0" $out/pytest.log && bash tools/final_measure.sh r2m
