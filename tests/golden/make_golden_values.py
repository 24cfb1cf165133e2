"""Golden fixtures for the per-token value quantization mode, from the
UNMODIFIED reference (run in the build container, where it is importable):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_values.py

Writes tests/golden/golden_values.npz: value matrices (including constant rows,
exact-half and large-range rows), quantize_uniform(PER_TOKEN, bits) codes,
zero points and scales (baseline_quant.py:69-110), the dequantized rows
(dequantize_uniform, :143-167) and PackedKVCache(quantize_values=True).values()
(kv_cache.py:199-209, 247-259).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main() -> None:
    import polarquant as pq  # the reference, read-only
    from polarquant.baseline_quant import QuantAxis, dequantize_uniform, quantize_uniform

    out: dict[str, np.ndarray] = {}
    for i, (T, bits, seed) in enumerate([(200, 4, 0), (64, 4, 1), (97, 2, 2), (33, 8, 3)]):
        rng = np.random.default_rng(seed)
        v = rng.standard_normal((T, 128)).astype(np.float32)
        v[3] = 0.5  # constant row -> scale 0
        v[5, :] = np.linspace(-1.0, 1.0, 128, dtype=np.float32)  # many exact halves
        v[7] *= 1e4
        v[9] = v[9].astype(np.float16).astype(np.float32)
        codes, params = quantize_uniform(v, bits, QuantAxis.PER_TOKEN)
        deq = dequantize_uniform(codes, params)
        keys = pq.gen_synthetic_keys(pq.SyntheticConfig(T, 128, seed=seed)).data
        cache = pq.PackedKVCache(pq.QuantConfig(4, 4), 0, quantize_values=True, value_bits=bits)
        cache.prefill(keys, v)
        out[f"v{i}/values"] = v
        out[f"v{i}/bits"] = np.array(bits)
        out[f"v{i}/codes"] = codes
        out[f"v{i}/zero_point"] = params.zero_point
        out[f"v{i}/scale"] = params.scale
        out[f"v{i}/dequant"] = deq
        out[f"v{i}/cache_values"] = cache.values()
    np.savez_compressed(HERE / "golden_values.npz", **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
