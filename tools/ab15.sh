export PYTHONUNBUFFERED=1
out=gpurun_out/ab15; mkdir -p $out
for i in 1 2; do
timeout 300 python bench.py --config 1 --no-cpu --no-e2e > $out/c1_graph_$i.json 2> $out/c1_graph.err
timeout 300 python bench.py --config 1 --no-cpu --no-e2e --no-graph > $out/c1_nograph_$i.json 2> $out/c1_nograph.err
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "config1 or small" > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
