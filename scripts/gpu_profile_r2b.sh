# Round-2 end-state ncu: the shipped G=4 / G=8 decode launches (grouped value
# layout, epilogue-count producers), the tcgen05 P.V A/B build, and the launch
# list of a 4-layer bench step.  CSV pages come back in gpurun_out/r2b/.
mkdir -p gpurun_out/r2b /tmp/r2b
NCU="ncu --clock-control none"
export_rep() {
  ncu -i /tmp/r2b/$1.ncu-rep --page raw --csv > gpurun_out/r2b/$1_raw.csv 2>/dev/null
  ncu -i /tmp/r2b/$1.ncu-rep --page details --csv > gpurun_out/r2b/$1_details.csv 2>/dev/null
}
for spec in "bf16 g4" "bf16 g8"; do
  set -- $spec
  timeout 600 $NCU --set full --import-source on -k regex:decode_dq -s 3 -c 1 -o /tmp/r2b/dq_$1_$2 -f python scripts/decode_probe.py $1 2 $2 > /dev/null 2>&1
  echo "ncu dq $1 $2 rc=$?"; export_rep dq_$1_$2
done
PQB_LIB=build_ab/libpqb200_umma_rel.so timeout 600 $NCU --set full -k regex:decode_dq -s 3 -c 1 -o /tmp/r2b/dq_umma_g4 -f python scripts/decode_probe.py bf16 2 g4 > /dev/null 2>&1
echo "ncu umma rc=$?"; export_rep dq_umma_g4
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2b/launches.csv python bench.py --profile --layers 4 --steps 2 --no-cpu --no-extras > /dev/null 2>&1; echo "launch list rc=$?"
du -sh gpurun_out
