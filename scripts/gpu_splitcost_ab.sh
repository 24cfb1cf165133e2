# PQB_SPLIT_COST A/B on the final build: headline bench alternating 24 (default) / 12 / 36
mkdir -p gpurun_out
for i in 1 2; do
  for c in 24 12 36; do
    sleep 4
    PQB_SPLIT_COST=$c python bench.py --no-extras --no-parity --no-cpu > gpurun_out/sc_${c}_${i}.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/sc_${c}_${i}.json')); print('cost $c rep $i', round(d['value']), round(d['sustained']['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"
  done
done
