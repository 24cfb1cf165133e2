# DQ kernel: parity tests, full decode tests, LUT-vs-DQ probe.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -x -k "dq" -p no:cacheprovider > gpurun_out/test_dq.log 2>&1; echo "dq tests rc=$?"; tail -30 gpurun_out/test_dq.log
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider > gpurun_out/test_gpu_decode.log 2>&1; echo "decode tests rc=$?"; tail -5 gpurun_out/test_gpu_decode.log
timeout 900 python scripts/dq_probe.py > gpurun_out/dq_probe.json 2> gpurun_out/dq_probe.err; echo "probe rc=$?"; cat gpurun_out/dq_probe.json; tail -5 gpurun_out/dq_probe.err
