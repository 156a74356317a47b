mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c43_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c43_smoke.log
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/c43_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c43_pytest.log
timeout 900 python bench.py > gpurun_out/c43_bench_C4.json 2> gpurun_out/c43_bench_C4.err
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 > gpurun_out/c43_bench_$C.json 2> gpurun_out/c43_bench_$C.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c43_launches_C3.csv python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c43_ncu_C3.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c43_launches_C4.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c43_ncu_C4.log 2>&1
echo done
