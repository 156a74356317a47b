mkdir -p gpurun_out
(cd scripts/probes && timeout 120 ./jacobi_probe jacobi_G_C2.txt > ../../gpurun_out/c22_jacobi.log 2>&1)
timeout 600 python -m pytest tests/test_gpu_parity_r2.py -x -q -m gpu -k "hot or sync_free or multi_window" > gpurun_out/c22_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c22_pytest.log
for C in C2 C3; do
  timeout 600 python scripts/diag_opts.py $C '{"rhs_hot_rows": 0}' '{"rhs_hot_rows": -1}' >> gpurun_out/c22_opts.log 2>&1
done
timeout 900 python scripts/diag_opts.py C4 '{"rhs_hot_rows": 0}' '{"rhs_hot_rows": -1}' >> gpurun_out/c22_opts.log 2>&1
echo done
