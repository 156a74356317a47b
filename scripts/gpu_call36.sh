mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c36_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c36_pytest.log
timeout 900 python scripts/create_timing.py C4 > gpurun_out/c36_create.json 2> gpurun_out/c36_create.err
timeout 900 python bench.py > gpurun_out/c36_bench_C4.json 2> gpurun_out/c36_bench_C4.err
echo done
