mkdir -p gpurun_out
for lib in paper_2006_16438_b200/libcparls.so build_variants/*.so; do
  CPARLS_LIB=$PWD/$lib timeout 600 python scripts/diag_variants.py C4 >> gpurun_out/c19_variants.log 2>> gpurun_out/c19_variants.err
done
echo done
