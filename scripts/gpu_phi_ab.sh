# A/B: G = 8 P.V with / without the P_lo MMA (ab/lib_a.so default, ab/lib_b.so PQB_DQ_PHI_ONLY=1)
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in a b; do sleep 5; PQB_LIB=ab/lib_$v.so python scripts/g8_rate.py $v$i 2>&1 | tail -1; done
done
python - <<'PY'
import torch
a, b = torch.load("gpurun_out/g8_out_a1.pt"), torch.load("gpurun_out/g8_out_b1.pt")
print("max|a-b|", (a - b).abs().max().item(), "max|a|", a.abs().max().item())
PY
