mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c33_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c33_smoke.log
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/c33_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c33_pytest.log
timeout 900 python bench.py > gpurun_out/c33_bench_C4.json 2> gpurun_out/c33_bench_C4.err
for C in C2 C3; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c33_bench_$C.json 2> gpurun_out/c33_bench_$C.err
done
echo done
