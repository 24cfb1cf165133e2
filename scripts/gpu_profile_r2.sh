# Round-2 ncu evidence: full captures of the shipped decode variants and the
# encoder, plus the launch list of a 4-layer bench step.  Full reports stay in
# /tmp/r2 on the box (too large to return); their raw / details / source
# pages come back as CSV in gpurun_out/r2/ (summaries go to profiles/r02/).
mkdir -p gpurun_out/r2 /tmp/r2
NCU="ncu --clock-control none"
export_rep() {  # $1 = report stem
  ncu -i /tmp/r2/$1.ncu-rep --page raw --csv > gpurun_out/r2/$1_raw.csv 2>/dev/null
  ncu -i /tmp/r2/$1.ncu-rep --page details --csv > gpurun_out/r2/$1_details.csv 2>/dev/null
  ncu -i /tmp/r2/$1.ncu-rep --page source --csv --print-source sass > /tmp/r2/$1_sass.csv 2>/dev/null
  gzip -c /tmp/r2/$1_sass.csv > gpurun_out/r2/$1_sass.csv.gz
}
for spec in ${SPECS:-"bf16 g4" "bf16 g8" "bf16 m3n2" "vq4 g4" "f32 g4" "vq8 g4"}; do
  set -- $spec
  timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o /tmp/r2/dq_$1_$2 -f python scripts/decode_probe.py $1 2 $2 > /dev/null 2>&1
  echo "ncu dq $1 $2 rc=$?"; export_rep dq_$1_$2
done
if [ -z "$SPECS" ]; then
timeout 600 $NCU --set full --import-source on -k regex:encode_fast -s 2 -c 1 -o /tmp/r2/encode_fast -f python scripts/encode_probe.py > /dev/null 2>&1; echo "ncu enc rc=$?"; export_rep encode_fast
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2/launches.csv python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
fi
du -sh gpurun_out
