mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_create_host.py -x -q > gpurun_out/c50_create_host.log 2>&1; echo "rc=$?" >> gpurun_out/c50_create_host.log
timeout 600 python scripts/create_timing.py C4 > gpurun_out/c50_create_timing.json 2> gpurun_out/c50_create_timing.err
timeout 900 python bench.py --config C4 > gpurun_out/c50_bench_C4.json 2> gpurun_out/c50_bench_C4.err; echo "rc=$?" >> gpurun_out/c50_bench_C4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c50_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c50_smoke.log
echo done
