mkdir -p gpurun_out/vq
timeout 600 ncu --clock-control none --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o /tmp/vq4 -f env PQB_LIB=${VQLIB:-paper_2502_00527_b200/libpqb200.so} python scripts/decode_probe.py vq4 2 g4 > /dev/null 2>&1
echo "ncu rc=$?"
ncu -i /tmp/vq4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -c > gpurun_out/vq/vq4_sass.csv.gz
ncu -i /tmp/vq4.ncu-rep --page raw --csv > gpurun_out/vq/vq4_raw.csv 2>/dev/null
