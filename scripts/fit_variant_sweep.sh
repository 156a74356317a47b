# Fit-kernel variant sweep (experiments): bench each libcparls_<v>.so given as arguments.
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="CPARLS_LIB=paper_2006_16438_b200/libcparls_$v.so"; fi
  env $L python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fv_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/fv_{v}.json"))
print(v, round(d["value"], 3), round(d["kernels"]["k_fit_sub"]["avg_ms"], 2), round(d["kernels"]["k_rhs"]["avg_ms"], 3))
PY
done
