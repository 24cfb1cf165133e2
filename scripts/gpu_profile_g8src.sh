# ncu full capture (source counters) of the configs[3]-shaped G=8 cluster launch with the bf16-P instance
mkdir -p gpurun_out/r2d /tmp/r2d
timeout 900 ncu --clock-control none --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o /tmp/r2d/dq_g8_bf16p -f python scripts/decode_probe.py bf16 2 g8 > /dev/null 2>&1
echo "ncu rc=$?"
ncu -i /tmp/r2d/dq_g8_bf16p.ncu-rep --page raw --csv > gpurun_out/r2d/dq_g8_bf16p_raw.csv 2>/dev/null
ncu -i /tmp/r2d/dq_g8_bf16p.ncu-rep --page details --csv > gpurun_out/r2d/dq_g8_bf16p_details.csv 2>/dev/null
ncu -i /tmp/r2d/dq_g8_bf16p.ncu-rep --page source --csv --print-source sass > gpurun_out/r2d/dq_g8_bf16p_sass.csv 2>/dev/null
cp /tmp/r2d/dq_g8_bf16p.ncu-rep gpurun_out/r2d/
ls -la gpurun_out/r2d
