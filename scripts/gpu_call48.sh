mkdir -p gpurun_out
timeout 900 python scripts/fit_overlap_ab.py C4 20 > gpurun_out/c48_ab_C4.json 2> gpurun_out/c48_ab_C4.err
timeout 600 python scripts/fit_overlap_ab.py C3 50 > gpurun_out/c48_ab_C3.json 2> gpurun_out/c48_ab_C3.err
echo done
