mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c30_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c30_pytest.log
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c30_bench_$C.json 2> gpurun_out/c30_bench_$C.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c30_warm_C2.csv python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c30_ncu_C2.log 2>&1
echo done
