"""Golden fixtures for the element-wise API, the synthetic generator and the
container formats, made by running the UNMODIFIED reference package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_api.py

Writes tests/golden/golden_api.npz:
  syn{i}/{cfg,keys}            gen_synthetic_keys (tensor_core.py:226-241)
  polar_{f32,f64}/{x,y,r,t}    to_polar (polar_codec.py:200-209)
  qa_{f32,f64}/{theta,codes}   quantize_angle for m = 1..8 (polar_codec.py:212-221)
  grid/m{m}                    angle_grid (polar_codec.py:224-233)
  qr{i}/{radius,scale,bits,codes,clamped}   quantize_radius / _quantize_radius_counted
  pqc/{blob}                   save_codes bytes of a reference cache's codes
  snap/{blob,after_angle,after_radius,after_residual,after_clamps,app_keys}
                               save_snapshot bytes, and the reference's
                               load_snapshot(...) state after two appends
  direct/{cfg,keys,q,scores}   qk_scores_direct of a reference cache
"""

from __future__ import annotations

import math
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main() -> None:
    import polarquant as pq  # the reference, read-only
    from numpy._core._multiarray_umath import __cpu_features__

    out: dict[str, np.ndarray] = {}

    def add(name: str, **arrays) -> None:
        for k, v in arrays.items():
            out[f"{name}/{k}"] = np.asarray(v)

    # ---- synthetic generator (per-channel means, outliers, both layouts)
    syn = [
        dict(num_tokens=64, dim=16, seed=3),
        dict(num_tokens=50, dim=128, seed=11, outlier_channels=frozenset({0, 1}), layout=pq.PairingLayout.ADJACENT),
        dict(num_tokens=33, dim=8, seed=7, radius_log_mean=np.array([0.0, 0.5, -1.0, 2.0]),
             radius_log_std=np.array([0.1, 0.5, 1.0, 0.0]), outlier_channels=frozenset({2}), outlier_log_boost=1.5),
    ]
    for i, kw in enumerate(syn):
        cfg = pq.SyntheticConfig(**kw)
        add(f"syn{i}", keys=pq.gen_synthetic_keys(cfg).data,
            mean=cfg.radius_log_mean, std=cfg.radius_log_std,
            meta=np.array([cfg.num_tokens, cfg.dim, cfg.seed, cfg.layout.value], np.int64),
            outliers=np.array(sorted(cfg.outlier_channels), np.int64), boost=np.float64(cfg.outlier_log_boost))

    # ---- to_polar: float32 (numpy SIMD arctan2) and float64 inputs, with the
    # wrap (-1, 0), the origin and axis points
    rng = np.random.default_rng(1234)
    edge = np.array([[-1.0, 0.0], [0.0, 0.0], [0.0, 2.0], [3.0, 4.0], [-0.0, -1.0], [1e-30, -1e-30], [-5.0, -0.0]])
    for name, dt in (("f32", np.float32), ("f64", np.float64)):
        x = np.concatenate([edge[:, 0], rng.standard_normal(4000) * 3]).astype(dt)
        y = np.concatenate([edge[:, 1], rng.standard_normal(4000) * 3]).astype(dt)
        r, t = pq.to_polar(x, y)
        assert r.dtype == dt and t.dtype == dt
        add(f"polar_{name}", x=x, y=y, r=r, t=t)

    # ---- quantize_angle: float64 (the reference tests' Python floats) and float32
    th64 = np.concatenate([[0.0, math.pi / 4, 3 * math.pi / 4, 1.5 * math.pi, 2 * math.pi - 1e-9, 2 * math.pi,
                            -0.3, 7.0], rng.uniform(0, 2 * math.pi, 5000)])
    th32 = np.concatenate([np.float32([0.0, np.pi / 4, 2 * np.pi, 6.2831855, -1.0]),
                           rng.uniform(0, 2 * math.pi, 5000).astype(np.float32)])
    add("qa_f64", theta=th64, codes=np.stack([pq.quantize_angle(th64, m) for m in range(1, 9)]))
    add("qa_f32", theta=th32, codes=np.stack([pq.quantize_angle(th32, m) for m in range(1, 9)]))
    for m in range(1, 9):
        out[f"grid/m{m}"] = pq.angle_grid(m)

    # ---- quantize_radius: float32 radii x per-channel scales (with zero scales,
    # clamps), float64 radii x a scalar scale
    radii = rng.uniform(0, 40, (300, 6)).astype(np.float32)
    scales = np.float16(radii.max(axis=0) / 3).astype(np.float32)
    scales[2] = 0.0
    scales[4] *= 0.5  # clamps
    for i, (rad, sc, bits) in enumerate([(radii, scales, 2), (radii, scales, 4), (radii.astype(np.float64), np.float32(1.7), 3),
                                         (np.float32(9.9), np.float32(1.0), 2)]):
        codes = pq.quantize_radius(rad, sc, bits)
        from polarquant.polar_codec import _quantize_radius_counted

        _, clamped = _quantize_radius_counted(np.asarray(rad), np.asarray(sc), bits)
        add(f"qr{i}", radius=rad, scale=sc, bits=np.int64(bits), codes=codes, clamped=np.int64(clamped))

    # ---- PQC1 and snapshot containers of a reference cache
    keys = pq.gen_synthetic_keys(pq.SyntheticConfig(40, 16, seed=5)).data
    cache = pq.PackedKVCache(pq.QuantConfig(5, 3, pq.PairingLayout.ADJACENT), 4)
    cache.prefill(keys)
    for row in pq.gen_synthetic_keys(pq.SyntheticConfig(6, 16, seed=8)).data:
        cache.append(row)
    with tempfile.TemporaryDirectory() as tmp:
        p = Path(tmp) / "c.pqc"
        snap = cache.snapshot()
        pq.save_codes(snap.codes, snap.scales, p)
        add("pqc", blob=np.frombuffer(p.read_bytes(), np.uint8))
        s = Path(tmp) / "c.snap"
        pq.save_snapshot(cache, s)
        add("snap", blob=np.frombuffer(s.read_bytes(), np.uint8))
        loaded = pq.load_snapshot(s)
        app = pq.gen_synthetic_keys(pq.SyntheticConfig(2, 16, seed=9)).data * 3.0
        for row in app:
            loaded.append(row)
        q = loaded.quantized
        add("snap", app_keys=app, after_angle=np.frombuffer(q.angle_stream, np.uint8),
            after_radius=np.frombuffer(q.radius_stream, np.uint8), after_residual=loaded.residual_keys,
            after_clamps=np.int64(loaded.clamp_events), after_tokens=np.int64(loaded.num_tokens))

    # ---- qk_scores_direct
    dk = pq.gen_synthetic_keys(pq.SyntheticConfig(500, 128, seed=21, outlier_channels=frozenset({0}))).data
    dc = pq.PackedKVCache(pq.QuantConfig(4, 3), 16)
    dc.prefill(dk)
    dq = rng.standard_normal(128).astype(np.float32)
    add("direct", keys=dk, q=dq, cfg=np.array([4, 3, 1, 16], np.int64), scores=pq.qk_scores_direct(dq, dc),
        lut=pq.qk_scores(dq, dc))

    out["__cpu_features__"] = np.array(sorted(k for k, v in __cpu_features__.items() if v))
    out["__numpy__"] = np.array(np.__version__)
    np.savez_compressed(HERE / "golden_api.npz", **out)
    print(f"wrote {len(out)} arrays to {HERE / 'golden_api.npz'}")


if __name__ == "__main__":
    main()
