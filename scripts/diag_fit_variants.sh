# exact-fit kernel time on C4 for library variants (CPARLS_LIB) of the L2 hint budgets
mkdir -p gpurun_out
for lib in build_variants/*.so; do
  echo "== $lib" >> gpurun_out/c6_fitvar.log
  CPARLS_LIB=$PWD/$lib timeout 600 python scripts/diag_fit.py -1 >> gpurun_out/c6_fitvar.log 2>> gpurun_out/c6_fitvar.err
done
echo done
