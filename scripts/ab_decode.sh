# A/B of two library builds (ab/lib_a.so, ab/lib_b.so): alternate processes with cool-down
for i in 1 2 3; do
  for v in a b; do sleep 6; echo -n "$v: "; PQB_LIB=ab/lib_$v.so python scripts/decode_rate.py; done
done
