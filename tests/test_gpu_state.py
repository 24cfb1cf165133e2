"""Cache state machine under growth and faults (advisor findings, round 1):
views survive pool growth, a non-finite key does not poison later appends,
a failed prefill resets only its own units, and the linear-layout build of
the DQ kernel (the runtime fallback of the PRMT table layout) matches."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_2502_00527_b200 as pq
from paper_2502_00527_b200 import _lib
from oracle import exact, polar_oracle as po
from tests.helpers import peak_close

pytestmark = pytest.mark.gpu


def _ref_out(cache, u, q, vals64):
    a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
    s16 = cache.scales16[u].cpu().numpy()
    res = cache.residual_keys(u).cpu().numpy()
    T = int(cache.host_seq[u])
    sc = po.lut_scores(q, a, r, s16, cache.cfg.angle_bits, cache.cfg.radius_bits, 1, res if res.size else None)
    return po.softmax64(sc, 1.0 / math.sqrt(128)) @ vals64[:T]


def test_view_survives_growth():
    """A view built before an append past capacity re-derives its descriptor
    (the pool and page table were replaced) instead of reading freed memory."""
    U, T, extra = 3, 200, 80
    keys = np.stack([po.synthetic_keys(T, 128, seed=70 + u) for u in range(U)])
    rng = np.random.default_rng(3)
    vals = rng.standard_normal((U, T + extra, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 16, capacity=T, page_tokens=64,
                            value_dtype=torch.float32)
    cache.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals[:, :T]).cuda())
    view = cache.view(0, U)
    q = rng.standard_normal((U, 4, 128)).astype(np.float32)
    qd = torch.from_numpy(q).cuda()
    view.decode(qd)
    pool0 = cache.pool.data_ptr()
    for i in range(extra):
        k = rng.standard_normal((U, 128)).astype(np.float32)
        cache.append(torch.from_numpy(k).cuda(), torch.from_numpy(vals[:, T + i]).cuda())
    assert cache.pool.data_ptr() != pool0, "the test must grow the pool"
    del pool0
    torch.cuda.empty_cache()
    got = view.decode(qd).cpu().numpy()
    v64 = vals.astype(np.float64)
    for u in range(U):
        for g in range(4):
            peak_close(got[u, g], _ref_out(cache, u, q[u, g], v64[u]), 1e-4)


def test_nonfinite_append_does_not_poison_cache():
    """Reference append does not validate keys (kv_cache.py:179-189): a NaN key
    is committed and later appends keep working; the batched cache's checked
    append raises for that call only."""
    cache = pq.PackedKVCache(pq.QuantConfig(4, 4), 2)
    cache.prefill(po.synthetic_keys(40, 16, seed=1))
    cache.append(np.full(16, np.nan, np.float32))
    for _ in range(4):
        cache.append(np.ones(16, np.float32))
    assert cache.num_tokens == 45
    b = pq.PolarKVCache(pq.QuantConfig(4, 4), 2, 128, 4, capacity=64)
    b.prefill(torch.from_numpy(np.stack([po.synthetic_keys(32, 128, seed=s) for s in (1, 2)])).cuda())
    bad = torch.full((2, 128), float("nan"), device="cuda")
    with pytest.raises(ValueError):
        b.append(bad, check=True)
    b.append(torch.ones(2, 128, device="cuda"), check=True)  # a fresh flag word per checked call
    b.append(bad)  # unchecked: recorded for check()
    with pytest.raises(ValueError):
        b.check()
    b.check()  # cleared
    q = pq.PackedKVCache(pq.QuantConfig(4, 4), 0, quantize_values=True)
    q.prefill(po.synthetic_keys(8, 16, seed=2))
    n0 = q.num_tokens
    with pytest.raises(ValueError):
        q.append(np.ones(16, np.float32), np.full(16, np.inf, np.float32))
    assert q.num_tokens == n0, "values are validated before anything is written"


def test_failed_prefill_resets_only_its_units():
    U, T = 4, 300
    keys = np.stack([po.synthetic_keys(T, 128, seed=30 + u) for u in range(U)])
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T, page_tokens=64, shuffle_pages=True)
    cache.prefill(torch.from_numpy(keys[:2]).cuda(), unit_start=0)
    bad = keys[2:].copy()
    bad[1, 17, 5] = np.nan
    with pytest.raises(ValueError):
        cache.prefill(torch.from_numpy(bad).cuda(), unit_start=2)
    assert cache._filled.tolist() == [True, True, False, False]
    cache.prefill(torch.from_numpy(keys[2:]).cuda(), unit_start=2)  # the units are fresh again
    for u in range(U):
        s16 = exact.scales(keys[u], 4, 1)
        ea, er, _ = exact.encode(keys[u], s16, 4, 4, 1)
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        assert np.array_equal(a, ea) and np.array_equal(r, er)


@pytest.mark.parametrize("m,n,G", [(4, 4, 4), (4, 4, 8), (3, 2, 4), (2, 4, 8)])
def test_dq_linear_layout_build(m, n, G):
    """PQB_DECODE_DQ_LINEAR runs the linear-layout build (decode_dq_lin.cu),
    the automatic fallback when the PRMT table placement does not fit."""
    U, T = 3, 3000
    keys = np.stack([po.synthetic_keys(T, 128, seed=400 + u, outliers=(0, 1)) for u in range(U)])
    rng = np.random.default_rng(11)
    vals = torch.from_numpy(rng.standard_normal((U, T, 128)).astype(np.float32)).to(torch.bfloat16)
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(m, n), U, 128, 0, capacity=T, page_tokens=128)
    cache.prefill(torch.from_numpy(keys).cuda(), vals.cuda())
    qd = torch.from_numpy(q).cuda()
    lin = cache._all().decode(qd, flags=_lib.PQB_DECODE_DQ | _lib.PQB_DECODE_DQ_LINEAR).cpu().numpy()
    dflt = cache._all().decode(qd, flags=_lib.PQB_DECODE_DQ).cpu().numpy()
    v64 = vals.float().numpy().astype(np.float64)
    for u in range(U):
        for g in range(G):
            ref = _ref_out(cache, u, q[u, g], v64[u])
            peak_close(lin[u, g], ref, 1e-4)
            peak_close(dflt[u, g], ref, 1e-4)
