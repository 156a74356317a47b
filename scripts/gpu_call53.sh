# Re-entry verification: smoke, full pytest -m gpu, default bench (C4) on the rebuilt library.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c53_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c53_smoke.log
timeout 1500 python bench.py > gpurun_out/c53_bench_C4.json 2> gpurun_out/c53_bench_C4.err
timeout 3000 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/c53_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c53_pytest.log
tail -3 gpurun_out/c53_smoke.log gpurun_out/c53_pytest.log; cat gpurun_out/c53_bench_C4.json
