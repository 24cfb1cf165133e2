# Round-1 final evidence: ncu captures of the shipped kernels, launch list,
# full GPU test suite, smoke, default bench.
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/r1f_decode_dq -f python scripts/decode_probe.py 0 2 g4 > /dev/null 2>&1; echo "dq rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/r1f_decode_dq_g8 -f python scripts/decode_probe.py 0 2 g8 > /dev/null 2>&1; echo "dq g8 rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:encode_fast -s 2 -c 1 -o gpurun_out/r1f_encode_fast -f python scripts/encode_probe.py > /dev/null 2>&1; echo "enc rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r1f_launches.csv python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
bash scripts/gpu_check.sh
timeout 300 python -m pytest tests/test_peer_gather.py -m gpu -q > gpurun_out/peer.log 2>&1; echo "peer rc=$?"; tail -2 gpurun_out/peer.log
