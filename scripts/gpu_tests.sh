# full GPU suite (+ optional extra command); logs in gpurun_out/
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/gpu_tests.log
