mkdir -p gpurun_out
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c20_bench_$C.json 2> gpurun_out/c20_bench_$C.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c20_launches_$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c20_ncu_$C.log 2>&1
done
echo done
