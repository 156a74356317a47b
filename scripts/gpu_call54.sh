# (1) k_rhs with the shared-memory hot-row set forced on C4 (first alternative);
# (2) launch list of HEAD's bench command (after it exited 0 without ncu).
mkdir -p gpurun_out
timeout 900 python scripts/diag_opts.py C4 '{}' '{"rhs_hot_rows": 1024}' '{"rhs_hot_rows": 256}' '{"rhs_hot_rows": 0}' > gpurun_out/c54_rhs_hot_C4.jsonl 2> gpurun_out/c54_rhs_hot_C4.err
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/c54_plain.json 2> gpurun_out/c54_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c54_launches_C4.csv $CMD > gpurun_out/c54_ncu1.log 2>&1
cat gpurun_out/c54_rhs_hot_C4.jsonl | cut -c1-600
echo done
