for w in 48 64 96 112; do
  CPARLS_RHS_WIN_MB=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/w$w.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/w'+sys.argv[1]+'.json')); print(sys.argv[1], round(d['value'],3), round(d['kernels']['k_rhs']['avg_ms'],3))" $w
done
