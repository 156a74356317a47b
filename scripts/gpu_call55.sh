# C2 / C3 bench lines of HEAD (secondary configs), after the re-entry rebuild.
mkdir -p gpurun_out
timeout 600 python bench.py --config C2 --no-e2e --no-cpu-baseline > gpurun_out/c55_bench_C2.json 2> gpurun_out/c55_bench_C2.err
timeout 600 python bench.py --config C3 --no-e2e --no-cpu-baseline > gpurun_out/c55_bench_C3.json 2> gpurun_out/c55_bench_C3.err
echo done
