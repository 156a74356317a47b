mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/c42_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c42_pytest.log
for C in C4 C3; do
timeout 600 python scripts/kernel_ab.py $C 10 > gpurun_out/c42_ab_pipe_$C.json 2> gpurun_out/c42_ab_pipe_$C.err
CPARLS_LIB=variants/libcparls_nopipe.so timeout 600 python scripts/kernel_ab.py $C 10 > gpurun_out/c42_ab_nopipe_$C.json 2> gpurun_out/c42_ab_nopipe_$C.err
done
echo done
