mkdir -p gpurun_out
timeout 900 python scripts/create_timing.py C4 > gpurun_out/c35_create.json 2> gpurun_out/c35_create.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c35_create_launches.csv python scripts/create_timing.py C3 > gpurun_out/c35_ncu.log 2>&1
echo done
