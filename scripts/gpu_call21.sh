mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c21_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c21_pytest.log
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c21_bench_$C.json 2> gpurun_out/c21_bench_$C.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c21_launches_C2.csv python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c21_ncu_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_krp_gram_t|k_rhs_hot|k_sidx_run|k_lookup|k_solve_prep|k_norm_prep" --launch-skip 40 --launch-count 12 -o gpurun_out/c21_full_C2 python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c21_ncufull_C2.log 2>&1
echo done
