# A/B: ab/lib_b.so vs ab/lib_a.so:
# headline bench (value median of 3 + 2.5 s sustained) alternating, then decode_rate (page 256)
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in a b; do
    sleep 5
    PQB_LIB=ab/lib_$v.so python bench.py --no-extras --no-parity --no-cpu > gpurun_out/ab_$v$i.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_$v$i.json')); print('$v$i', round(d['value']), round(d['sustained']['value']), d['clocks']['sm_mhz'], d['sustained']['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"
  done
done
for v in a b; do sleep 4; echo -n "$v: "; PQB_PAGE=256 PQB_LIB=ab/lib_$v.so python scripts/decode_rate.py 2>&1 | tail -1; done
