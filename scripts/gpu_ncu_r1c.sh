# ncu evidence for the round-1 final kernels (one GPU, single process)
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/r1c_decode_dq -f python scripts/decode_probe.py 0 2 > /dev/null 2>&1; echo "dq rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o gpurun_out/r1c_decode_dq_vq4 -f python scripts/decode_probe.py 4 2 > /dev/null 2>&1; echo "vq4 rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:encode_fast -s 2 -c 1 -o gpurun_out/r1c_encode_fast -f python scripts/encode_probe.py > /dev/null 2>&1; echo "enc rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:radius_max_tma -s 2 -c 1 -o gpurun_out/r1c_rmax -f python scripts/encode_probe.py > /dev/null 2>&1; echo "rmax rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r1c_launches.csv python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
ls -la gpurun_out | grep r1c
