export PYTHONUNBUFFERED=1
out=gpurun_out/ab9; mkdir -p $out
timeout 300 python tools/vcheck.py 4096 5 > $out/vcheck.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
bash tools/ab.sh -c 2 -r 3 variants/nosd.so paper_1301_0763_b200/libqftb200.so > $out/ab.log 2>&1
