set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
(cd scripts/probes && ./atomics_probe) > gpurun_out/c1_probe.log 2>&1
timeout 900 python scripts/diag_rhs_skew.py C4 3 > gpurun_out/c1_skew.json 2> gpurun_out/c1_skew.err
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c1_b.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed,lts__d_atomic_input_cycles_active.min.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red_lookup_hit.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.max.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,lts__t_sectors.max,lts__t_sectors.avg,lts__xbar2lts_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__xbar2lts_cycles_active.max.pct_of_peak_sustained_elapsed,lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput_internal_activity.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_rhs -s 3 -c 3 --csv --log-file gpurun_out/c1_ncu_rhs.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c1_ncu.log 2>&1
echo done
