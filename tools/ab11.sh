export PYTHONUNBUFFERED=1
out=gpurun_out/ab11; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k classical > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > $out/c4.json 2> $out/c4.err
