mkdir -p gpurun_out
(cd scripts/probes && timeout 120 ./jacobi_probe jacobi_G_C2.txt > ../../gpurun_out/c23_jacobi.log 2>&1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c23_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c23_pytest.log
for C in C2 C3; do
  timeout 600 python scripts/diag_opts.py $C '{"rhs_hot_rows": 0}' '{"rhs_hot_rows": -1}' >> gpurun_out/c23_opts.log 2>&1
done
timeout 900 python scripts/diag_opts.py C4 '{"rhs_hot_rows": 0}' '{"rhs_hot_rows": -1}' >> gpurun_out/c23_opts.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c23_launches_C2.csv python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c23_ncu_C2.log 2>&1
echo done
