mkdir -p gpurun_out
timeout 900 python scripts/create_timing.py C4 > gpurun_out/c41_create.json 2> gpurun_out/c41_create.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rhs|k_fit_sub|k_solve_dmma|k_lev_rows_w" --launch-skip 30 --launch-count 5 -o gpurun_out/c41_full_C4 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c41_ncufull_C4.log 2>&1
echo done
