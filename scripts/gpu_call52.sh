mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_create_host.py -x -q > gpurun_out/c52_create_host.log 2>&1; echo "rc=$?" >> gpurun_out/c52_create_host.log
timeout 900 python bench.py --config C4 > gpurun_out/c52_bench_C4.json 2> gpurun_out/c52_bench_C4.err; echo "rc=$?" >> gpurun_out/c52_bench_C4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c52_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c52_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c52_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/c52_pytest_gpu.log
echo done
