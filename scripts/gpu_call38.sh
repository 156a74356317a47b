mkdir -p gpurun_out
timeout 600 python scripts/fit_hot_sweep.py C4 0,256,448,1024 > gpurun_out/c38_sweep_pf0.log 2>&1
for v in 1 2 3; do
CPARLS_LIB=variants/libcparls_pf$v.so timeout 600 python scripts/fit_hot_sweep.py C4 0,448 > gpurun_out/c38_sweep_pf$v.log 2>&1
done
timeout 1800 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/c38_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c38_pytest.log
echo done
