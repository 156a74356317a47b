mkdir -p gpurun_out
python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c12_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -s 700 -c 600 --csv --log-file gpurun_out/c12_launches_C3.csv python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c12_ncu.log 2>&1
echo done
