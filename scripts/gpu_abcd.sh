# A/B/C/D over ab/lib_{a,b,c,d}.so: configs[3] shape (g8_rate) then the headline bench, alternating
mkdir -p gpurun_out
for i in 1 2; do
  for v in a b c d; do sleep 4; PQB_LIB=ab/lib_$v.so python scripts/g8_rate.py $v$i 2>&1 | tail -1; done
done
for i in 1 2; do
  for v in a b c d; do
    sleep 4
    PQB_LIB=ab/lib_$v.so python bench.py --no-extras --no-parity --no-cpu > gpurun_out/ab4_$v$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab4_$v$i.json')); print('$v$i', round(d['value']), round(d['sustained']['value']), d['clocks']['sm_mhz'])"
  done
done
