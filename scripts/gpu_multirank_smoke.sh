# The bench's N > 1 code paths as 2 ranks on ONE GPU over gloo (this
# environment has a single GPU): batch-sharded, KV-head-sharded with the fused
# peer gather and with the NCCL-path gather (eager: gloo collectives cannot be
# captured in a CUDA graph; NCCL ones can), and the reference arm.
set -x
export PQB_BENCH_BACKEND=gloo PQB_BENCH_DEVICE=0
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29511 bench.py --gpus 2 --layers 4 --steps 4 --warmup 3 --sustain-seconds 0 > gpurun_out/mr_batch.json 2> gpurun_out/mr_batch.err; echo "batch rc=$?"; tail -c 600 gpurun_out/mr_batch.json
timeout 600 $R --master-port 29512 bench.py --gpus 2 --layers 4 --steps 4 --warmup 3 --shard heads --sustain-seconds 0 > gpurun_out/mr_heads.json 2> gpurun_out/mr_heads.err; echo "heads p2p rc=$?"; tail -c 600 gpurun_out/mr_heads.json
timeout 600 $R --master-port 29513 bench.py --gpus 2 --layers 4 --steps 4 --warmup 3 --shard heads --gather nccl --no-graph --sustain-seconds 0 > gpurun_out/mr_heads_nccl.json 2> gpurun_out/mr_heads_nccl.err; echo "heads nccl-path rc=$?"; tail -c 300 gpurun_out/mr_heads_nccl.json
timeout 600 $R --master-port 29514 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 --cpu-seconds 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/mr_ref.json
