mkdir -p gpurun_out
(cd scripts/probes && ./atomics_probe) > gpurun_out/c7_probe.log 2>&1
echo done
