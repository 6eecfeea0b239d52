export PYTHONUNBUFFERED=1
out=gpurun_out/ab12; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_full_batch.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
bash tools/ab.sh -c 4 -r 2 variants/nostg.so paper_1301_0763_b200/libqftb200.so > $out/ab_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none \
    -k regex:"lg_f" -c 8 --csv --log-file $out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 1 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
rm -f variants/nostg.so
