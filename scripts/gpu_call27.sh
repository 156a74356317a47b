mkdir -p gpurun_out
timeout 600 python scripts/diag_fit_modes.py C3 >> gpurun_out/c27_fitmodes.log 2>&1
timeout 600 python scripts/diag_fit_modes.py C2 >> gpurun_out/c27_fitmodes.log 2>&1
for C in C2 C3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c27_warm_$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c27_ncu_$C.log 2>&1
done
echo done
