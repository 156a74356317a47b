mkdir -p gpurun_out
timeout 1500 python scripts/diag_fit.py -1 0 1 2 > gpurun_out/c4_fit.json 2> gpurun_out/c4_fit.err
echo done
