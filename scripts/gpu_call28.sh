mkdir -p gpurun_out
(cd scripts/probes && timeout 60 ./smallla_probe > ../../gpurun_out/c28_smallla.log 2>&1)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fit_sub" -c 1 -o gpurun_out/c28_fit_C3 python scripts/diag_fit_modes.py C3 > gpurun_out/c28_ncufit.log 2>&1
echo done
