mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_api.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2 3; do
  for lib in build_ab/lib_default.so build_ab/lib_sc8.so; do
    echo -n "$lib "; PQB_LIB=$lib timeout 300 python scripts/scores_rate.py 2>>gpurun_out/ab.err
  done
done
