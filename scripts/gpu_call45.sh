mkdir -p gpurun_out
timeout 600 python scripts/kernel_ab.py C4 10 > gpurun_out/c45_ab_async_C4.json 2> gpurun_out/c45_ab_async_C4.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c1_lockstep_20 or boundary or c5 or free_running" > gpurun_out/c45_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c45_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fit_async" -c 1 -o gpurun_out/c45_fit_async python scripts/kernel_ab.py C4 5 > gpurun_out/c45_ncu.log 2>&1
echo done
