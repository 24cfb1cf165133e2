# One gpurun pass: GPU parity tests (one pytest process per file so a device
# fault cannot poison the rest), smoke(), then a short bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
for f in tests/test_gpu_encode.py tests/test_gpu_decode.py tests/test_gpu_api.py; do
  [ -f "$f" ] || continue
  b=$(basename $f .py)
  timeout 900 python -m pytest "$f" -m gpu -q --maxfail=10 -p no:cacheprovider > gpurun_out/$b.log 2>&1; echo "$b rc=$?"
  tail -15 gpurun_out/$b.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 1200 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
if [ "${NCU_ENCODE:-0}" = "1" ]; then
  ncu --clock-control none --set full --import-source on -k regex:radius_max -s 2 -c 1 -o gpurun_out/rmax_latest -f python scripts/encode_probe.py > /dev/null 2>&1; echo "rmax ncu rc=$?"
fi
