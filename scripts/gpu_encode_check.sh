set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -m gpu -q --maxfail=5 -p no:cacheprovider > gpurun_out/test_gpu_encode.log 2>&1; echo "enc tests rc=$?"; tail -3 gpurun_out/test_gpu_encode.log
timeout 600 python -c "
import bench, torch, json
print(json.dumps(bench.encode_bench(torch.device('cuda',0), None)))
" > gpurun_out/encode_bench.json 2>&1; echo "enc bench rc=$?"; cat gpurun_out/encode_bench.json
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:encode_v8 -s 2 -c 1 -o gpurun_out/encode_v3 -f python scripts/encode_probe.py > /dev/null 2>&1; echo "encode ncu rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:radius_max_v8 -s 2 -c 1 -o gpurun_out/rmax_v3 -f python scripts/encode_probe.py > /dev/null 2>&1; echo "rmax ncu rc=$?"
