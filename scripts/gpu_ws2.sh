# Warp-split decode A/B: per-launch timing of library builds (alternating) + launch-phase traces.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest $TESTS -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gpu_tests.log; fi
LIBS=${LIBS:-"build_ab/libpqb200_head.so paper_2502_00527_b200/libpqb200.so build_ab/libpqb200_blk.so"}
for rep in 1 2; do
  for lib in $LIBS; do
    echo "== $lib"; PQB_LIB=$lib PQB_PAGE=256 timeout 300 python scripts/decode_rate.py 2>>gpurun_out/ab.err
  done
done
for s in g8 g4; do
  PQB_LIB=build_ab/libpqb200_trace.so timeout 300 python scripts/trace_probe.py $s 2>>gpurun_out/trace.err | tee gpurun_out/trace_$s.json
done
