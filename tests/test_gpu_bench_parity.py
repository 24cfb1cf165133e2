"""Parity at exactly the configurations bench.py times:
the bench's own DecodeWorkload (on-device Philox keys / values / queries,
page 256, bf16 q / V / out, the default kernel choice incl. the PRMT table
and the separate merge launch), one layer of each config, checked unit by unit
with oracle/parity.py: scales and codes bit-exact vs the correctly rounded C
oracle, ties vs the numpy restatement of the reference counted and admissible,
outputs within 2^-7 max|o| + 1 bf16 ulp of softmax64(LUT scores) . V.
Also the bench's N > 1 paths, run as 2 ranks on this box's GPU."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _run_layer(**spec):
    import torch

    import bench
    from paper_2502_00527_b200 import _lib

    keep = spec.pop("keep")
    flags = spec.pop("flags", 0)
    dev = torch.device("cuda", 0)
    w = bench.DecodeWorkload(dev, layers=1, page_tokens=256, seed=3, keep=keep, **spec)
    w.base_flags = flags
    run = w.capture(w.step)
    launches = int(_lib.load().pqb_decode_launches(w.upl, w.G, w.T, flags))
    summ = bench.parity_leg(w, keep, run)
    w.free()
    return summ, launches


def _assert_ok(summ, units):
    assert summ["units"] == units
    assert summ["scale_mismatches"] == 0
    assert summ["exact_code_mismatches"] == 0
    assert summ["non_tie_mismatches"] == 0, summ
    assert summ["tie_rate"] <= 1e-5, summ
    assert summ["out_within_tol"], summ
    assert summ["passed"]


def test_configs1_headline_layer_all_units():
    """configs[1]: 128 units x 32,768 tokens, m4n4, G = 4, DQ + PRMT, bf16 q/V/out."""
    summ, launches = _run_layer(batch=16, hq=32, hkv=8, T=32768, m=4, n=4, keep=list(range(128)))
    _assert_ok(summ, 128)
    assert launches == 1
    print(json.dumps({k: v for k, v in summ.items() if k != "cpu_features"}))


def test_configs2_m3n2_128k():
    """configs[2]: m3n2 at 131,072 tokens (64 units per layer; 12 sampled)."""
    summ, _ = _run_layer(batch=8, hq=32, hkv=8, T=131072, m=3, n=2, keep=[0, 5, 9, 17, 22, 30, 33, 41, 48, 55, 60, 63])
    _assert_ok(summ, 12)


def test_configs3_g8_cluster_merge():
    """configs[3] per GPU: G = 8, 32 units x 32,768 tokens; as benched, each unit
    runs on a 4-CTA thread-block cluster that merges through distributed shared
    memory (one launch)."""
    summ, launches = _run_layer(batch=32, hq=8, hkv=1, T=32768, m=4, n=4, keep=list(range(32)))
    _assert_ok(summ, 32)
    assert launches == 1


def test_configs3_g8_separate_merge():
    """configs[3] without the cluster path: balanced split, split merge in its own launch."""
    from paper_2502_00527_b200 import _lib

    summ, launches = _run_layer(batch=32, hq=8, hkv=1, T=32768, m=4, n=4, keep=list(range(32)),
                                flags=_lib.PQB_DECODE_NO_CLUSTER)
    _assert_ok(summ, 32)
    assert launches == 2


@pytest.mark.parametrize("values", ["vq2", "vq4", "vq8"])
def test_configs1_quantized_values(values):
    """The reference's per-token value quantization (kv_cache.py:199-209) at 2 / 4 / 8 bits."""
    summ, _ = _run_layer(batch=16, hq=32, hkv=8, T=32768, m=4, n=4, values=values, keep=[0, 7, 64, 127])
    _assert_ok(summ, 4)


def test_configs1_f32_values():
    """The reference's default value cache (fp32 rows, kv_cache.py:8-9, :209)."""
    summ, _ = _run_layer(batch=16, hq=32, hkv=8, T=32768, m=4, n=4, values="f32", keep=[0, 3, 66, 120])
    _assert_ok(summ, 4)


@pytest.mark.parametrize("shard", ["batch", "heads"])
def test_bench_two_ranks(shard):
    """``python bench.py --gpus 2`` spawns two ranks itself; both sharding
    modes print one line with n_gpus 2, e2e no faster than the device value,
    and a passing parity leg (the fused peer gather's outputs are checked)."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--layers", "2", "--ctx", "8192", "--steps", "4",
           "--warmup", "3", "--reps", "1", "--no-extras", "--no-cpu", "--sustain-seconds", "0", "--shard", shard,
           "--parity-sample", "4"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["parity"]["passed"] and d["parity"]["ranks"] == 2
    assert d["e2e"]["value"] <= d["value"] * 1.10  # host copies inside the timed region (noise allowance)


@pytest.mark.parametrize("values", ["bf16", "f32", "vq2", "vq4", "vq8"])
def test_fp32_outputs_at_32k(values):
    """fp32 outputs of the fused decode at the bench's context length for every
    value treatment: max |o - ref| <= 1e-4 max(1, max |ref|) against
    softmax64(LUT scores) . values() (the quantized modes remove their code
    offset per tile and split off the rows' midpoints, see decode_dq.cu)."""
    import math

    import numpy as np
    import torch

    import bench
    from oracle import exact, polar_oracle as po

    dev = torch.device("cuda", 0)
    keep = list(range(0, 128, 16))
    w = bench.DecodeWorkload(dev, layers=1, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=256, seed=7,
                             values=values, keep=keep)
    o32 = w.views[0].decode(w.q[0], out_dtype=torch.float32).cpu().numpy()
    for u in keep:
        _, vv = w.kept[u]
        v64 = (w.cache.values_f32(u) if values.startswith("vq") else vv.float()).cpu().numpy().astype(np.float64)
        a, r = (t.cpu().numpy() for t in w.cache.code_arrays(u))
        s16 = w.cache.scales16[u].cpu().numpy()
        q = w.q[0, u].float().cpu().numpy()
        for g in range(4):
            ref = po.softmax64(exact.lut_scores(q[g], a, r, s16, 4, 4, 1), 1 / math.sqrt(128)) @ v64
            assert np.abs(o32[u, g] - ref).max() <= 1e-4 * max(1.0, float(np.abs(ref).max()))
    w.free()
