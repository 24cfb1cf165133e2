# Cluster / DSMEM split-merge path: decode tests, then configs[3]-shaped per-layer timing with and
# without it (PQB_DECODE_NO_CLUSTER), alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python scripts/cluster_probe.py
