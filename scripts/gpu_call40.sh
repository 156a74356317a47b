mkdir -p gpurun_out
timeout 900 python scripts/fit_overlap_sweep.py C4 0,74,37,111,148 20 > gpurun_out/c40_overlap.log 2>&1
timeout 600 python scripts/fit_overlap_sweep.py C3 0,74 50 > gpurun_out/c40_overlap_C3.log 2>&1
echo done
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -x -q -m gpu -k "overlapped or recovers or sync_free or boundary" > gpurun_out/c40_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c40_pytest.log
