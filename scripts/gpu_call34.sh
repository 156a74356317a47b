mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_red_probe scripts/probes/tma_red_probe.cu && timeout 300 /tmp/tma_red_probe > gpurun_out/c34_tma_probe.log 2>&1
echo "rc=$?" >> gpurun_out/c34_tma_probe.log
timeout 600 python scripts/degree_skew.py > gpurun_out/c34_skew.json 2> gpurun_out/c34_skew.err
echo done
