"""Small invocations of every shipped kernel, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck; scripts/gpu_sanitize.sh).

    python scripts/sanitize.py [case ...]     (default: all cases)

Sizes are tiny (sanitizers serialise and instrument every access) but each
case still takes the production code path: multi-CTA splits with the
last-CTA merge and the separate merge launch, PRMT table layout, producer
warpgroup, 4-bit values, residual window, streaming append."""

from __future__ import annotations

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2502_00527_b200 as pq  # noqa: E402
from paper_2502_00527_b200 import _lib  # noqa: E402


def _cache(m, n, U, T, *, res=0, vb=None, vdt=torch.bfloat16, page=256, seed=1):
    syn = pq.SyntheticConfig(T, 128, outlier_channels=frozenset({0, 1}))
    keys = pq.synthetic_keys_device(syn, U, dtype=torch.bfloat16, seed=seed)
    vals = pq.normal_device((U, T, 128), seed + 1, dtype=torch.bfloat16)
    c = pq.PolarKVCache(pq.QuantConfig(m, n), U, 128, res, capacity=T + 64, page_tokens=page, value_dtype=vdt,
                        value_bits=vb)
    c.prefill(keys, vals)
    return c


def case_encode():
    for m, n in [(4, 4), (3, 2), (2, 4)]:
        _cache(m, n, 2, 4096)
    # generic encoder / K1 (d = 64, fp32 keys, ADJACENT)
    k = torch.randn(3, 1000, 64, device="cuda")
    c = pq.PolarKVCache(pq.QuantConfig(5, 3, pq.PairingLayout.ADJACENT), 3, 64, 0, capacity=1000, page_tokens=64,
                        value_dtype=torch.float32)
    c.prefill(k)


def case_decode_g4():
    c = _cache(4, 4, 4, 8192)
    q = pq.normal_device((4, 4, 128), 5, dtype=torch.bfloat16)
    c.decode(q, out_dtype=torch.bfloat16)
    c._all().decode(q, flags=_lib.PQB_DECODE_MERGE_KERNEL)


def case_decode_g8():
    c = _cache(4, 4, 2, 20000)
    q = pq.normal_device((2, 8, 128), 6, dtype=torch.bfloat16)
    c.decode(q, out_dtype=torch.bfloat16)
    c._all().decode(q, flags=_lib.PQB_DECODE_MERGE_KERNEL)


def case_decode_m3n2():
    c = _cache(3, 2, 3, 5000)
    q = pq.normal_device((3, 4, 128), 7, dtype=torch.bfloat16)
    c.decode(q, out_dtype=torch.bfloat16)


def case_decode_cluster():
    # 32 units of G = 8: the thread-block-cluster path (4 CTAs per unit, DSMEM merge)
    c = _cache(4, 4, 32, 8192)
    q = pq.normal_device((32, 8, 128), 21, dtype=torch.bfloat16)
    a = c.decode(q)
    b = c.decode(q, flags=pq._lib.PQB_DECODE_NO_CLUSTER)
    torch.cuda.synchronize()
    print("cluster vs no-cluster max abs diff", (a - b).abs().max().item())


def case_decode_vq4():
    c = _cache(4, 4, 3, 4096, vb=4)
    q = pq.normal_device((3, 4, 128), 8, dtype=torch.bfloat16)
    c.decode(q)


def case_decode_vq28():
    for vb in (2, 8):
        c = _cache(4, 4, 3, 4096, vb=vb)
        q = pq.normal_device((3, 4, 128), 12, dtype=torch.bfloat16)
        c.decode(q)
        c = _cache(3, 2, 2, 3000, vb=vb)
        q = pq.normal_device((2, 8, 128), 13, dtype=torch.bfloat16)
        c.decode(q)


def case_decode_f32v():
    c = _cache(4, 4, 3, 4096, vdt=torch.float32)
    q = pq.normal_device((3, 4, 128), 9, dtype=torch.bfloat16)
    c.decode(q)


def case_scores():
    c = _cache(4, 4, 2, 3000)
    q = pq.normal_device((2, 4, 128), 10, dtype=torch.float32)
    c.scores(q)
    c._all().scores(q, flags=_lib.PQB_DECODE_DQ)
    c._all().decode(q, flags=_lib.PQB_DECODE_LUT)


def case_append_residual():
    c = _cache(4, 4, 2, 1000, res=32, page=128)
    q = pq.normal_device((2, 4, 128), 11, dtype=torch.float32)
    for i in range(40):
        c.append(torch.randn(2, 128, device="cuda"), torch.randn(2, 128, device="cuda"))
    c.decode(q)
    c.scores(q)


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        torch.cuda.synchronize()
        print(f"case {name}: ok", flush=True)
