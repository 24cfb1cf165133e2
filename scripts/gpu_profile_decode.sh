set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --import-source on -k regex:decode_fast -s 3 -c 1 -o gpurun_out/decode_v2 -f \
  python bench.py --profile --layers 2 --steps 3 --no-encode --no-cpu > gpurun_out/ncu_decode_v2.log 2>&1; echo "decode ncu rc=$?"
tail -3 gpurun_out/ncu_decode_v2.log
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/launches_v2.csv \
  python bench.py --profile --layers 4 --steps 2 --no-encode --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
