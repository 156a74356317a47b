mkdir -p gpurun_out
(cd scripts/probes && ./atomics_probe) > gpurun_out/c2_probe.log 2>&1
timeout 1200 python scripts/diag_rhs_skew.py C4 3 > gpurun_out/c2_skew.json 2> gpurun_out/c2_skew.err
echo done
