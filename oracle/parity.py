"""Parity of sampled cache units against the oracles -- TEST INFRASTRUCTURE ONLY.

Used by the -m gpu parity tests (tests/test_gpu_bench_parity.py) and by
bench.py's parity leg, which runs after the timed region on units sampled
from the very caches the benchmark timed.  The product package never imports
this module.  Per unit:

  * scales  bit-identical to the correctly rounded C restatement
            (exact_oracle.c, pinned to the reference's fixtures);
  * codes   bit-identical to the C restatement, and compared with the numpy
            restatement of the reference (oracle/polar_oracle.py, the
            reference's own float32 numpy sequence): every difference must be
            an admissible tie (angle within 4 ulp(pi_f32) of a bin edge,
            radius within 2^-20 of a rounding boundary); ties are counted;
  * output  softmax64(LUT scores of the unit's codes) . V in float64 vs the
            GPU's output, |err| <= rtol * max|o| + atol (bf16 output:
            rtol = 2^-7 plus one bf16 ulp of max|o|; fp32: 1e-4).

The float64 softmax . V over the GPU codes is the restated reference output
(the reference stops at the weights, lut_decode.py:189-206).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from oracle import exact, polar_oracle as po

BF16_RTOL = 2.0**-7
F32_RTOL = 1e-4


def cpu_features() -> list[str]:
    from numpy._core._multiarray_umath import __cpu_features__

    return sorted(k for k, v in __cpu_features__.items() if v)


@dataclass
class UnitResult:
    scale_mismatch: int = 0
    exact_mismatch: int = 0          # vs the correctly rounded C oracle (must be 0)
    numpy_angle_mismatch: int = 0    # vs the numpy reference sequence
    numpy_radius_mismatch: int = 0
    non_tie: int = 0                 # numpy mismatches that are not admissible ties (must be 0)
    codes: int = 0
    out_err: float = 0.0             # max |o - ref| / max(1, max |ref|)
    out_excess: float = 0.0          # max (|o - ref| - bound), <= 0 when inside the tolerance
    notes: list = field(default_factory=list)


def check_unit(keys: np.ndarray, s16_gpu: np.ndarray, angle_gpu: np.ndarray, radius_gpu: np.ndarray, m: int, n: int,
               layout: int = po.HALF_SPLIT, *, q: np.ndarray | None = None, values: np.ndarray | None = None,
               out: np.ndarray | None = None, sm_scale: float | None = None, out_bf16: bool = True,
               numpy_ties: bool = True) -> UnitResult:
    """keys (T, d) float32 (exactly what the GPU encoded); codes (T, d/2) uint8
    read back from the GPU cache; q (G, d), values (T, d) float32 (what the GPU
    stored), out (G, d) the GPU output as float32."""
    res = UnitResult()
    keys = np.ascontiguousarray(keys, dtype=np.float32)
    T, d = keys.shape
    s16 = exact.scales(keys, n, layout)
    res.scale_mismatch = int(np.count_nonzero(s16.view(np.uint16) != np.asarray(s16_gpu, np.float16).view(np.uint16)))
    ea, er, _ = exact.encode(keys, s16, m, n, layout)
    res.codes = int(ea.size)
    res.exact_mismatch = int(np.count_nonzero(ea != angle_gpu) + np.count_nonzero(er != radius_gpu))
    if numpy_ties:
        na, nr, _ = po.encode_block(keys, s16, m, n, layout)
        am, rm = na != angle_gpu, nr != radius_gpu
        res.numpy_angle_mismatch = int(am.sum())
        res.numpy_radius_mismatch = int(rm.sum())
        if am.any() or rm.any():
            x, y = po.split_xy(keys, layout)
            ok_a = po.classify_angle_mismatch(x[am], y[am], m) | rm[am]
            s32 = np.broadcast_to(s16.astype(np.float32), x.shape)
            ok_r = po.radius_tie(x[rm], y[rm], s32[rm])
            res.non_tie = int((~ok_a).sum() + (~ok_r).sum())
    if q is not None and out is not None and values is not None:
        scale = (1.0 / math.sqrt(d)) if sm_scale is None else sm_scale
        v64 = np.asarray(values, np.float64)
        worst, excess = 0.0, -np.inf
        for g in range(q.shape[0]):
            sc = exact.lut_scores(q[g], angle_gpu, radius_gpu, s16, m, n, layout)
            ref = po.softmax64(sc, scale) @ v64
            peak = float(np.abs(ref).max())
            err = float(np.abs(np.asarray(out[g], np.float64) - ref).max())
            bound = (BF16_RTOL * peak + float(np.spacing(np.float32(peak))) * 2.0**16 if out_bf16
                     else F32_RTOL * max(1.0, peak))  # bf16 ulp = 2^16 f32 ulps
            worst = max(worst, err / max(1.0, peak))
            excess = max(excess, err - bound)
        res.out_err, res.out_excess = worst, excess
    return res


def summarize(results: list[UnitResult]) -> dict:
    codes = sum(r.codes for r in results)
    ties = sum(r.numpy_angle_mismatch + r.numpy_radius_mismatch for r in results)
    return {
        "units": len(results),
        "codes_checked": codes,
        "scale_mismatches": sum(r.scale_mismatch for r in results),
        "exact_code_mismatches": sum(r.exact_mismatch for r in results),
        "numpy_ties": ties,
        "numpy_angle_ties": sum(r.numpy_angle_mismatch for r in results),
        "numpy_radius_ties": sum(r.numpy_radius_mismatch for r in results),
        "tie_rate": ties / codes if codes else 0.0,
        "non_tie_mismatches": sum(r.non_tie for r in results),
        "max_out_rel_err": max((r.out_err for r in results), default=0.0),
        "out_within_tol": all(r.out_excess <= 0 for r in results),
        "cpu_features": cpu_features(),
        "numpy": np.__version__,
    }


def passed(summary: dict) -> bool:
    return (summary["scale_mismatches"] == 0 and summary["exact_code_mismatches"] == 0
            and summary["non_tie_mismatches"] == 0 and summary["out_within_tol"]
            and summary["tie_rate"] <= 1e-5)


def check_many(jobs, threads: int = 0) -> list[UnitResult]:
    """jobs: iterable of kwargs for check_unit; run on host threads (numpy and
    the ctypes oracle release the GIL)."""
    import os

    jobs = list(jobs)
    n = threads or min(len(jobs), max(1, len(os.sched_getaffinity(0))))
    if n <= 1:
        return [check_unit(**j) for j in jobs]
    with ThreadPoolExecutor(max_workers=n) as ex:
        return list(ex.map(lambda j: check_unit(**j), jobs))
