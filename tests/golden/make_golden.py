"""Generate golden fixtures by running the UNMODIFIED reference package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Each case stores its inputs and the
reference's outputs (scales, packed streams, unpacked codes, clamp counts, LUT
scores, float64 attention weights and the restated softmax.V) plus the host's
numpy CPU features, because numpy's float32 arctan2 is dispatch-dependent.
The reference is only available in the build container; the fixtures travel.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main() -> None:
    import polarquant as pq  # the reference, read-only
    from numpy._core._multiarray_umath import __cpu_features__

    cases: dict[str, np.ndarray] = {}
    meta = []

    def add(name: str, **arrays) -> None:
        for k, v in arrays.items():
            cases[f"{name}/{k}"] = np.asarray(v)

    layouts = {0: pq.PairingLayout.ADJACENT, 1: pq.PairingLayout.HALF_SPLIT}

    # ---- encoder cases: synthetic keys through encode_keys / compute_radius_scales
    enc_cases = [
        (256, 128, 4, 4, 1, 0, 0),  # (T, d, m, n, layout, unused, seed)
        (300, 128, 3, 2, 1, 16, 1),
        (257, 128, 2, 2, 0, 0, 2),
        (200, 128, 2, 4, 1, 0, 3),
        (128, 128, 4, 2, 0, 0, 4),
        (96, 128, 8, 8, 1, 0, 5),
        (77, 64, 6, 3, 1, 0, 6),
        (50, 32, 5, 7, 0, 0, 7),
        (37, 10, 3, 5, 1, 0, 8),
        (40, 16, 1, 1, 1, 0, 9),
        (33, 2, 7, 6, 0, 0, 10),
        (64, 256, 4, 4, 1, 0, 11),
    ]
    for i, (T, d, m, n, lay, _res, seed) in enumerate(enc_cases):
        keys = pq.gen_synthetic_keys(
            pq.SyntheticConfig(T, d, seed=seed, layout=layouts[lay], outlier_channels=frozenset({0}) if d >= 4 else frozenset())
        ).data
        if i % 3 == 0:  # dead channel, tiny radii, exact zeros
            keys = keys.copy()
            half = d // 2
            x, y = pq.split_pairs(keys, layouts[lay])
            x[:, half - 1] = 0.0
            y[:, half - 1] = 0.0
            x[: T // 4] *= 1e-3
            y[: T // 4] *= 1e-3
        cfg = pq.QuantConfig(m, n, layouts[lay])
        scales = pq.compute_radius_scales(keys, cfg)
        codes = pq.encode_keys(keys, scales, cfg)
        x, y = pq.split_pairs(keys, layouts[lay])
        _, _, clamped = pq.polar_codec.quantize_subvectors(x, y, scales, cfg)
        add(f"enc{i}", keys=keys, cfg=np.array([T, d, m, n, lay]), scales=scales.values.view(np.uint16),
            angle_stream=np.frombuffer(codes.angle_stream, np.uint8), radius_stream=np.frombuffer(codes.radius_stream, np.uint8),
            angle=codes.angle_codes(), radius=codes.radius_codes(), clamped=np.array(clamped))
        meta.append(f"enc{i}")

    # ---- KATs from the reference tests (test_polar_codec.py / SURVEY 8(c))
    kat = np.array([[3, 4, 0, 0, 1e-4, 0, -1, 0], [0, 2, 0, 0, 2, 0, 0, -1]], dtype=np.float32)
    cfg = pq.QuantConfig(4, 4, pq.PairingLayout.ADJACENT)
    s = pq.compute_radius_scales(kat, cfg)
    c = pq.encode_keys(kat, s, cfg)
    add("kat_adjacent", keys=kat, scales=s.values.view(np.uint16), angle=c.angle_codes(), radius=c.radius_codes())

    # ---- cache cases: prefill + appends + scores + weights + softmax.V
    cache_cases = [
        (1024, 128, 4, 4, 1, 0, 100, 4),   # config-1 head shape (G=4 queries)
        (1000, 128, 3, 2, 1, 16, 101, 4),
        (700, 128, 2, 2, 0, 5, 102, 1),
        (300, 32, 4, 4, 1, 3, 103, 2),
        (129, 128, 4, 2, 1, 128, 104, 8),
        (40, 16, 5, 3, 0, 0, 105, 1),
    ]
    for i, (T, d, m, n, lay, res, seed, G) in enumerate(cache_cases):
        rng = np.random.default_rng([seed, 1])
        keys = pq.gen_synthetic_keys(pq.SyntheticConfig(T, d, seed=seed, layout=layouts[lay],
                                                        outlier_channels=frozenset({0, 1}))).data
        values = rng.standard_normal((T, d)).astype(np.float32)
        app_k = pq.gen_synthetic_keys(pq.SyntheticConfig(6, d, seed=seed + 1, layout=layouts[lay])).data * 1.5
        app_v = rng.standard_normal((6, d)).astype(np.float32)
        queries = rng.standard_normal((G, d)).astype(np.float32)
        cfg = pq.QuantConfig(m, n, layouts[lay])
        cache = pq.PackedKVCache(cfg, res)
        cache.prefill(keys, values)
        pre_scores = np.stack([pq.qk_scores(q, cache) for q in queries])
        for r_k, r_v in zip(app_k, app_v):
            cache.append(r_k, r_v)
        angle, radius = cache.code_arrays()
        scores = np.stack([pq.qk_scores(q, cache) for q in queries])
        temp = 1.0 / np.sqrt(d)
        weights = np.stack([pq.attention_weights(sc, temp) for sc in scores])
        out = weights @ cache.values().astype(np.float64)
        snap = cache.quantized
        add(f"cache{i}", keys=keys, values=values, app_keys=app_k, app_values=app_v, queries=queries,
            cfg=np.array([T, d, m, n, lay, res]), scales=cache.scales.values.view(np.uint16),
            pre_scores=pre_scores, scores=scores, weights=weights, out=out,
            angle_stream=np.frombuffer(snap.angle_stream, np.uint8),
            radius_stream=np.frombuffer(snap.radius_stream, np.uint8),
            clamps=np.array(cache.clamp_events), residual_keys=cache.residual_keys,
            radius_table=cache.radius_table(), decoded=cache.decode_quantized()[:64])
        meta.append(f"cache{i}")

    # ---- angle tables and query LUTs for every m
    for m in range(1, 9):
        t = pq.build_angle_table(m)
        q = np.random.default_rng(m).standard_normal(16).astype(np.float32)
        lut = pq.build_query_lut(q, t, pq.PairingLayout.HALF_SPLIT)
        add(f"table{m}", cos=t.cos, sin=t.sin, q=q, lut=lut.partial)

    cases["__cpu_features__"] = np.array([k for k, v in __cpu_features__.items() if v])
    cases["__numpy__"] = np.array(np.__version__)
    np.savez_compressed(HERE / "golden.npz", **cases)
    print(f"wrote {HERE / 'golden.npz'} ({len(meta)} cases)")


if __name__ == "__main__":
    sys.path.insert(0, "/root/reference/pkg/src")
    main()
