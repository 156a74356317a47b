mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/c17_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c17_pytest.log
timeout 1200 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c17_bench_C4.json 2> gpurun_out/c17_bench_C4.err
timeout 900 python bench.py --config C3 --no-e2e --no-cpu-baseline > gpurun_out/c17_bench_C3.json 2> gpurun_out/c17_bench_C3.err
echo done
