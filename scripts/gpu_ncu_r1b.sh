# ncu evidence for the transposed-QK decode kernel and the encoder (one GPU, single process)
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/decode_dq_t -f \
  python bench.py --profile --layers 2 --steps 3 --no-cpu --no-extras > gpurun_out/ncu_decode_dq_t.log 2>&1; echo "decode ncu rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:encode_v8 -s 2 -c 1 -o gpurun_out/encode_v8 -f \
  python scripts/encode_probe.py > gpurun_out/ncu_encode.log 2>&1; echo "encode ncu rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:radius_max -s 2 -c 1 -o gpurun_out/rmax -f \
  python scripts/encode_probe.py > gpurun_out/ncu_rmax.log 2>&1; echo "rmax ncu rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/launches_dq_t.csv \
  python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
ls -la gpurun_out
