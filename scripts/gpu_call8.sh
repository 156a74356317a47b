mkdir -p gpurun_out
rm -f gpurun_out/solve_bars.jsonl
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_sharded.py -x -q -m gpu --durations=15 > gpurun_out/c8_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c8_pytest.log
echo done
