mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c49_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_create_host.py -x -q > gpurun_out/c49_create_host.log 2>&1; echo "rc=$?" >> gpurun_out/c49_create_host.log
timeout 900 python bench.py --config C4 > gpurun_out/c49_bench_C4.json 2> gpurun_out/c49_bench_C4.err; echo "rc=$?" >> gpurun_out/c49_bench_C4.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c49_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/c49_pytest_gpu.log
echo done
