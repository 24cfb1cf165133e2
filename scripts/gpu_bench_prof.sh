set -x
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:encode_v8 -s 2 -c 1 -o gpurun_out/encode_v2 -f \
  python scripts/encode_probe.py > gpurun_out/ncu_encode_v2.log 2>&1; echo "encode ncu rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:radius_max_v8 -s 2 -c 1 -o gpurun_out/rmax_v2 -f \
  python scripts/encode_probe.py > gpurun_out/ncu_rmax_v2.log 2>&1; echo "rmax ncu rc=$?"
