# Final-build ncu: the shipped G=4 / G=8 decode launches (bf16-P instances, one QK chain,
# whole-tile softmax) and the launch list of a 4-layer bench step.  Reports in gpurun_out/r2f/.
mkdir -p gpurun_out/r2f
NCU="ncu --clock-control none"
for g in g4 g8; do
  timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/r2f/dq_bf16_$g -f python scripts/decode_probe.py bf16 2 $g > /dev/null 2>&1
  echo "ncu dq $g rc=$?"
done
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2f/launches_bench_4layers.csv python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
du -sh gpurun_out/r2f
