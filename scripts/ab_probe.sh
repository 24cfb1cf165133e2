# A/B timing of library builds (LIBS, space separated; default: previous commit vs current), alternating.
mkdir -p gpurun_out
LIBS=${LIBS:-"build_ab/libpqb200_head.so paper_2502_00527_b200/libpqb200.so"}
for rep in 1 2; do
  for lib in $LIBS; do
    echo "== $lib rep $rep"
    PQB_LIB=$lib timeout 600 python scripts/dq_probe.py "$@" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items():
    if isinstance(v,dict): print(k, 'frac', v['frac'], 'launch_ms', v['avg_launch_ms'])
"
  done
done
