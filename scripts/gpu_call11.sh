mkdir -p gpurun_out
rm -f gpurun_out/solve_bars.jsonl
timeout 3000 python -m pytest tests -x -q -m gpu --durations=20 > gpurun_out/c11_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c11_pytest.log
timeout 900 python bench.py --config C2 --no-e2e --no-cpu-baseline > gpurun_out/c11_bench_C2.json 2> gpurun_out/c11_bench_C2.err
timeout 900 python bench.py --config C3 --no-e2e --no-cpu-baseline > gpurun_out/c11_bench_C3.json 2> gpurun_out/c11_bench_C3.err
timeout 1200 python bench.py > gpurun_out/c11_bench_C4.json 2> gpurun_out/c11_bench_C4.err
echo done
