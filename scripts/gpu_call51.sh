mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_create_host.py -x -q > gpurun_out/c51_create_host.log 2>&1; echo "rc=$?" >> gpurun_out/c51_create_host.log
timeout 900 python bench.py --config C4 > gpurun_out/c51_bench_C4.json 2> gpurun_out/c51_bench_C4.err; echo "rc=$?" >> gpurun_out/c51_bench_C4.err
echo done
