# Microbenchmarks + encoder tests + encode bench (one gpurun call).
set -x
mkdir -p gpurun_out
timeout 120 ./scripts/micro/mma_rate > gpurun_out/micro.txt 2>&1; echo "micro rc=$?"; cat gpurun_out/micro.txt
timeout 900 python -m pytest tests/test_gpu_encode.py -m gpu -q --maxfail=5 -p no:cacheprovider > gpurun_out/test_gpu_encode.log 2>&1; echo "enc tests rc=$?"; tail -3 gpurun_out/test_gpu_encode.log
timeout 600 python -c "
import bench, torch, json
print(json.dumps(bench.encode_bench(torch.device('cuda',0), None)))
" > gpurun_out/encode_bench.json 2>&1; echo "enc bench rc=$?"; cat gpurun_out/encode_bench.json
