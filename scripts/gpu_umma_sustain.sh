# Sustained A/B (bench.py's 2.5 s back-to-back leg) of the default build vs the tcgen05 P.V build.
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in build_ab/lib_default.so build_ab/libpqb200_umma_rel.so; do
    sleep 5
    PQB_LIB=$lib timeout 600 python bench.py --no-extras --no-cpu --no-parity --reps 1 > gpurun_out/sus_$(basename $lib .so)_$rep.json 2>>gpurun_out/sus.err
    python - "$lib" gpurun_out/sus_$(basename $lib .so)_$rep.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(d["value"],1), "kernel_frac", round(d["roofline"]["frac"],3), "step_frac", round(d["roofline"]["step_frac"],3),
      "sustained", round(d["sustained"]["value"],1), "sus_mhz", d["sustained"]["clocks"]["sm_mhz"], d["sustained"]["clocks"]["reasons"])
PY
  done
done
