# Encoder A/B (configs[4] slab K1 + K2 times), alternating library builds; encoder tests first.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_encode.py tests/test_gpu_reference_api.py tests/test_gpu_api.py -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
for rep in 1 2 3; do
  for lib in ${LIBS:-build_ab/lib_default.so build_ab/lib_enc.so}; do
    echo -n "$lib: "; PQB_LIB=$lib timeout 300 python scripts/encode_timing.py 2>>gpurun_out/ab.err
  done
done
