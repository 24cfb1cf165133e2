# ncu full capture of the configs[3]-shaped G=8 decode launch on the cluster path, plus its launch list.
mkdir -p gpurun_out/r2c /tmp/r2c
timeout 600 ncu --clock-control none --set full -k regex:decode_dq -s 3 -c 1 -o /tmp/r2c/dq_g8_cluster -f python scripts/decode_probe.py bf16 2 g8 > /dev/null 2>&1
echo "ncu rc=$?"
ncu -i /tmp/r2c/dq_g8_cluster.ncu-rep --page raw --csv > gpurun_out/r2c/dq_g8_cluster_raw.csv 2>/dev/null
ncu -i /tmp/r2c/dq_g8_cluster.ncu-rep --page details --csv > gpurun_out/r2c/dq_g8_cluster_details.csv 2>/dev/null
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__cluster_dim_x --csv --log-file gpurun_out/r2c/launches_g8.csv python scripts/decode_probe.py bf16 4 g8 > /dev/null 2>&1
echo "launches rc=$?"
