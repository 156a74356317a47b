mkdir -p gpurun_out
timeout 600 python scripts/kernel_ab.py C4 10 > gpurun_out/c44_ab_async_C4.json 2> gpurun_out/c44_ab_async_C4.err
CPARLS_LIB=variants/libcparls_noasync.so timeout 600 python scripts/kernel_ab.py C4 10 > gpurun_out/c44_ab_noasync_C4.json 2> gpurun_out/c44_ab_noasync_C4.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c44_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c44_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "fit_against" > gpurun_out/c44_pytest_full.log 2>&1
echo "rc=$?" >> gpurun_out/c44_pytest_full.log
echo done
