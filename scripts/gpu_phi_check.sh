# bf16-P (G = 8, bf16 outputs) build: A/B against the previous build, decode GPU tests, configs[3] parity leg
mkdir -p gpurun_out
for i in 1 2; do
  for v in a b; do sleep 5; PQB_LIB=ab/lib_$v.so python scripts/g8_rate.py $v$i 2>&1 | tail -1; done
done
python - <<'PY'
import torch
a, b = torch.load("gpurun_out/g8_out_a1.pt"), torch.load("gpurun_out/g8_out_b1.pt")
print("max|a-b|", (a - b).abs().max().item(), "max|a|", a.abs().max().item())
PY
timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_parity.py tests/test_peer_gather.py tests/test_gpu_api.py -x -q -m gpu -p no:cacheprovider > gpurun_out/phi_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/phi_tests.log
