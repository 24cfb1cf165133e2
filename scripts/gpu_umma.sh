# tcgen05 P.V variant (PQB_DQ_UMMA build): parity tests on it, then per-launch A/B against the default build.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
PQB_LIB=${ULIB:-build_ab/libpqb200_umma.so} timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -p no:cacheprovider  > gpurun_out/umma_tests.log 2>&1; echo "umma pytest rc=$?"; tail -15 gpurun_out/umma_tests.log
LIBS=${LIBS:-"build_ab/libpqb200_head.so build_ab/lib_default.so build_ab/libpqb200_umma.so"}
for rep in 1 2; do
  for lib in $LIBS; do
    echo "== $lib"; PQB_LIB=$lib PQB_PAGE=256 timeout 300 python scripts/decode_rate.py 2>>gpurun_out/ab.err
  done
done
