# Sustained A/B (bench.py value + 2.5 s back-to-back leg; configs[1] bf16 and 4-bit values) of spinning vs
# sleeping mbarrier waits.
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in build_ab/lib_spin.so build_ab/lib_sleep_both.so; do
    for vals in bf16 vq4; do
      sleep 5
      PQB_LIB=$lib timeout 600 python bench.py --no-extras --no-cpu --no-parity --reps 3 --values $vals --sustain-seconds 4 > gpurun_out/sl.json 2>>gpurun_out/sl.err
      python - "$lib" "$vals" gpurun_out/sl.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], sys.argv[2], "value", round(d["value"],1), "sustained", round(d["sustained"]["value"],1), "mhz", d["sustained"]["clocks"]["sm_mhz"], "kernel", round(d["roofline"]["frac"],3))
PY
    done
  done
done
