# Launch-phase traces of the G=8 (configs[3]) and G=4 (configs[1]) decode launches
# and the G=8 fixed-cost scaling, on one box.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for s in g8 g4; do
  PQB_LIB=build_ab/libpqb200_trace.so timeout 300 python scripts/trace_probe.py $s 2>>gpurun_out/trace.err | tee gpurun_out/trace_$s.json
done
timeout 600 python scripts/g8_scaling.py 2>>gpurun_out/trace.err | tee gpurun_out/g8_scaling.json
