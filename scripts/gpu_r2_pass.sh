# Round-2 pass as the driver runs it: full GPU suite, smoke(), default bench,
# reference arm, and a 2-rank self-spawned bench (one GPU, two ranks).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -3 gpurun_out/bench_ref.err
if [ "${MULTI:-1}" = "1" ]; then
timeout 900 python bench.py --gpus 2 --no-cpu > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; echo "g2 rc=$?"; tail -3 gpurun_out/bench_g2.err
fi
