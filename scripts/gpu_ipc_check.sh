# Peer-gather buffers on pqb_ipc_alloc / pqb_ipc_open: the two-rank tests, the
# multi-rank bench smoke (batch / heads p2p / heads nccl) and the self-spawned
# 2-rank bench (its configs[2]/[3] KV-head-sharded lines use the fused gather).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_peer_gather.py tests/test_sharding.py tests/test_abi.py -x -q -m gpu -p no:cacheprovider > gpurun_out/ipc_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ipc_tests.log
bash scripts/gpu_multirank_smoke.sh > gpurun_out/ipc_mr.log 2>&1; grep "rc=" gpurun_out/ipc_mr.log
timeout 900 python bench.py --gpus 2 --no-cpu > gpurun_out/ipc_g2.json 2> gpurun_out/ipc_g2.err; echo "g2 rc=$?"; tail -3 gpurun_out/ipc_g2.err
