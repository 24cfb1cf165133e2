mkdir -p gpurun_out
PQB_LIB=build_ab/lib_2ch.so timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -p no:cacheprovider -k "vq" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
  for lib in build_ab/lib_default.so build_ab/lib_2ch.so; do
    echo "== $lib"; PQB_LIB=$lib PQB_PAGE=256 timeout 300 python scripts/decode_rate.py 2>>gpurun_out/ab.err
  done
done
