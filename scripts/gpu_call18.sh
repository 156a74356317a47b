mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/c18_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c18_pytest.log
timeout 1500 python bench.py > gpurun_out/c18_bench_C4.json 2> gpurun_out/c18_bench_C4.err
echo done
