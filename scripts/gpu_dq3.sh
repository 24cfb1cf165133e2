set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -p no:cacheprovider > gpurun_out/test_gpu_decode.log 2>&1; echo "decode tests rc=$?"; tail -4 gpurun_out/test_gpu_decode.log; grep -E "Error: max" gpurun_out/test_gpu_decode.log | head
LIBS="build_ab/libpqb200_head.so paper_2502_00527_b200/libpqb200.so" bash scripts/ab_probe.sh lut,dq G4_cfg1,G8_cfg3
