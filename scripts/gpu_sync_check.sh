mkdir -p gpurun_out/san
for c in decode_cluster decode_g4 decode_g8 decode_vq4 decode_f32v scores; do
  for tool in synccheck memcheck; do
    timeout 600 compute-sanitizer --print-limit 5 --error-exitcode 9 --tool $tool python scripts/sanitize.py $c > gpurun_out/san/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/san/${tool}_$c.log | tail -1)"
  done
done
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
