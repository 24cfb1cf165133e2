# configs[1] bench (value + 2.5 s sustained) with the persistent grid at 148 (default) vs 128 CTAs (one unit each).
mkdir -p gpurun_out
for rep in 1 2; do
  for n in 0 128; do
    sleep 5
    PQB_DQ_CTAS=$n timeout 600 python bench.py --no-extras --no-cpu --no-parity --reps 3 > gpurun_out/ctas_$n_$rep.json 2>>gpurun_out/ctas.err
    python - "$n" gpurun_out/ctas_$n_$rep.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print("ctas", sys.argv[1] or "148", "value", round(d["value"],1), d["value_reps"]["min"].__round__(1), d["value_reps"]["max"].__round__(1), "kernel", round(d["roofline"]["frac"],3), "step", round(d["roofline"]["step_frac"],3),
      "sustained", round(d["sustained"]["value"],1), d["sustained"]["clocks"]["sm_mhz"])
PY
  done
done
