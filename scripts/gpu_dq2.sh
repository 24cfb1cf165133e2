set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -k "dq" -p no:cacheprovider > gpurun_out/test_dq.log 2>&1; echo "dq tests rc=$?"; tail -4 gpurun_out/test_dq.log
timeout 900 python scripts/dq_probe.py > gpurun_out/dq_probe.json 2> gpurun_out/dq_probe.err; echo "probe rc=$?"; cat gpurun_out/dq_probe.json; tail -5 gpurun_out/dq_probe.err
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/dq_g4 -f \
  python bench.py --profile --layers 2 --steps 3 --variant dq --no-cpu --no-extras > gpurun_out/ncu_dq_g4.log 2>&1; echo "ncu g4 rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/dq_g8 -f \
  python bench.py --profile --layers 2 --steps 3 --hq 8 --hkv 1 --batch 32 --no-cpu --no-extras > gpurun_out/ncu_dq_g8.log 2>&1; echo "ncu g8 rc=$?"
