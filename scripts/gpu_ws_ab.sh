# A/B: warp-specialised decode (ab/lib_a.so) vs lane-0 issue (ab/lib_b.so)
set -x
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -m gpu > gpurun_out/ws_t_dec.log 2>&1; tail -3 gpurun_out/ws_t_dec.log
export PQB_PAGE=256
for i in 1 2 3; do
  for v in a b; do sleep 5; echo -n "$v: "; PQB_LIB=ab/lib_$v.so timeout 120 python scripts/decode_rate.py; done
done
for v in a b a b; do sleep 8; PQB_LIB=ab/lib_$v.so timeout 120 python scripts/sustain_probe.py | tail -1; done
