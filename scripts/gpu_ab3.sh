# A/B of library builds listed in $LIBS (ab/lib_X.so), burst decode rates, 3 rounds
set -x
[ "${RUN_TESTS:-1}" = "1" ] && { timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -m gpu > gpurun_out/ab_t_dec.log 2>&1; tail -2 gpurun_out/ab_t_dec.log; }
export PQB_PAGE=256
for i in 1 2 3; do
  for v in ${LIBS:-a b}; do sleep 5; echo -n "$v: "; PQB_LIB=ab/lib_$v.so timeout 120 python scripts/decode_rate.py; done
done
