mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/c32_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c32_pytest.log
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c32_bench_$C.json 2> gpurun_out/c32_bench_$C.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c32_warm_C3.csv python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c32_ncu_C3.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c32_bench_C4.json 2> gpurun_out/c32_bench_C4.err
echo done
