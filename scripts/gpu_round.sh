# Full round pass: GPU tests + smoke + bench, then the decode ncu evidence
# (one --set full capture of the headline kernel + the launch list of a short bench).
set -x
mkdir -p gpurun_out
SKIP_BENCH=0 bash scripts/gpu_check.sh
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/decode_dq_full -f \
  python bench.py --profile --layers 2 --steps 3 --no-cpu --no-extras > gpurun_out/ncu_decode_dq.log 2>&1; echo "ncu full rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/launches_dq.csv python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
