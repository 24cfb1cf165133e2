# ncu captures (one GPU, single process): full set on the top decode and encode
# kernels, plus the per-launch duration list of a short bench step.
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --import-source on -k regex:decode_fast -s 3 -c 1 -o gpurun_out/decode_full -f \
  python bench.py --profile --layers 2 --steps 3 --no-encode --no-cpu > gpurun_out/ncu_decode.log 2>&1; echo "decode ncu rc=$?"
tail -3 gpurun_out/ncu_decode.log
timeout 600 $NCU --set full --import-source on -k regex:encode_v8 -s 2 -c 1 -o gpurun_out/encode_full -f \
  python scripts/encode_probe.py > gpurun_out/ncu_encode.log 2>&1; echo "encode ncu rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:radius_max_v8 -s 2 -c 1 -o gpurun_out/rmax_full -f \
  python scripts/encode_probe.py > gpurun_out/ncu_rmax.log 2>&1; echo "rmax ncu rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile --layers 4 --steps 2 --no-encode --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
ls -la gpurun_out
