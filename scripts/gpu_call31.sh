mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/c31_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c31_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c31_bench_C4.json 2> gpurun_out/c31_bench_C4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rhs_hot|k_lookup|k_sidx_run|k_krp_rows|k_gram_rows_t|k_cand_count" --launch-skip 30 --launch-count 12 -o gpurun_out/c31_full_C3 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c31_ncufull_C3.log 2>&1
echo done
