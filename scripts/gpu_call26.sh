mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c26_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c26_pytest.log
timeout 600 python scripts/diag_opts.py C2 '{}' '{"fit_samples": 134217728, "fit_seed": 7}' >> gpurun_out/c26_opts.log 2>&1
timeout 600 python scripts/diag_opts.py C3 '{}' >> gpurun_out/c26_opts.log 2>&1
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c26_bench_$C.json 2> gpurun_out/c26_bench_$C.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c26_launches_$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c26_ncu_$C.log 2>&1
done
echo done
