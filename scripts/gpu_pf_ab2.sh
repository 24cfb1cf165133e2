# L2 page prefetch A/B: ab/lib_a (off), b (1 page), c (2), d (4) on the configs[3] shape, then decode_rate (page 256)
mkdir -p gpurun_out
for i in 1 2; do
  for v in a b c d; do sleep 4; PQB_LIB=ab/lib_$v.so python scripts/g8_rate.py $v$i 2>&1 | tail -1; done
done
for v in a c d; do sleep 4; echo -n "$v: "; PQB_PAGE=256 PQB_LIB=ab/lib_$v.so python scripts/decode_rate.py 2>&1 | tail -1; done
