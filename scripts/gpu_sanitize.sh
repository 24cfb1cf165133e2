# compute-sanitizer over every shipped kernel (scripts/sanitize.py cases) and
# the two-rank peer gather; logs in gpurun_out/san/.
mkdir -p gpurun_out/san
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
CASES="encode decode_g4 decode_g8 decode_m3n2 decode_vq4 decode_vq28 decode_f32v scores append_residual"
for tool in memcheck synccheck racecheck; do
  for c in $CASES; do
    timeout 900 $CS --tool $tool python scripts/sanitize.py $c > gpurun_out/san/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${c}.log | tail -1)"
  done
done
timeout 900 $CS --tool memcheck --target-processes all python -m pytest tests/test_peer_gather.py -m gpu -q -x > gpurun_out/san/memcheck_peer.log 2>&1
echo "memcheck peer rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san/memcheck_peer.log | tail -2 | tr '\n' ' ')"
