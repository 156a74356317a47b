mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c47_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c47_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "sampling" > gpurun_out/c47_pytest_full.log 2>&1
echo "rc=$?" >> gpurun_out/c47_pytest_full.log
for C in C3 C2; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c47_bench_$C.json 2> gpurun_out/c47_bench_$C.err
done
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c47_bench_C4.json 2> gpurun_out/c47_bench_C4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c47_launches_C3.csv python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c47_ncu_C3.log 2>&1
echo done
