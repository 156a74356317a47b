mkdir -p gpurun_out
timeout 1500 python scripts/diag_rhs_skew.py C4 3 > gpurun_out/c3_skew.json 2> gpurun_out/c3_skew.err
echo done
