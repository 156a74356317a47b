mkdir -p gpurun_out
for C in C3 C2; do timeout 600 python scripts/fit_overlap_ab.py $C 50 > gpurun_out/c46_ab_$C.json 2> gpurun_out/c46_ab_$C.err; done
timeout 900 python scripts/fit_overlap_ab.py C4 20 > gpurun_out/c46_ab_C4.json 2> gpurun_out/c46_ab_C4.err
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -x -q -m gpu -k "overlapped or recovers or sync_free or degrees" > gpurun_out/c46_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c46_pytest.log
echo done
