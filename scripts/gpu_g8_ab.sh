# configs[3]-shape A/B over library builds ab/lib_{a,b,c}.so (alternating processes)
mkdir -p gpurun_out
for i in 1 2; do
  for v in ${VARIANTS:-a b c}; do sleep 5; PQB_LIB=ab/lib_$v.so python scripts/g8_rate.py $v$i 2>&1 | tail -1; done
done
