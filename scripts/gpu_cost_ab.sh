# Balanced-split segment cost A/B (PQB_SPLIT_COST, 0 = uniform ranges), alternating, decode_rate shapes.
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest $TESTS -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log; fi
for rep in 1 2 3; do
  for c in ${COSTS:-0 16 24 32}; do
    echo -n "cost $c: "; PQB_SPLIT_COST=$c PQB_PAGE=256 timeout 300 python scripts/decode_rate.py 2>>gpurun_out/ab.err
  done
done
