mkdir -p gpurun_out
timeout 900 python scripts/fit_hot_sweep.py C4 0,128,256,448,1024 > gpurun_out/c37_sweep.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/c37_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c37_pytest.log
echo done
