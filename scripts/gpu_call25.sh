mkdir -p gpurun_out
(cd scripts/probes && timeout 120 ./jacobi_probe jacobi_G_C2.txt > ../../gpurun_out/c25_jacobi.log 2>&1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c25_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c25_pytest.log
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c25_bench_$C.json 2> gpurun_out/c25_bench_$C.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c25_launches_$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c25_ncu_$C.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_krp_gram_t|k_gram_scales|k_norm_prep|k_solve_prep|k_lookup|k_sidx_run|k_cand" --launch-skip 60 --launch-count 14 -o gpurun_out/c25_full_C3 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c25_ncufull_C3.log 2>&1
echo done
