"""Shared comparison helpers for the parity tests (test infrastructure)."""

from __future__ import annotations

import numpy as np

from oracle import polar_oracle as po


def case(golden: dict, name: str) -> dict:
    pre = name + "/"
    return {k[len(pre):]: v for k, v in golden.items() if k.startswith(pre)}


def case_names(golden: dict, prefix: str) -> list[str]:
    return sorted({k.split("/")[0] for k in golden if k.startswith(prefix)}, key=lambda s: int(s[len(prefix):]))


def compare_codes(keys, layout, m, n, s16, got_a, got_r, ref_a, ref_r, *, exact: bool):
    """Angle/radius code parity.  exact=True: bit-identical.  Otherwise every
    mismatch must be an admissible bin-edge tie; returns counts."""
    x, y = po.split_xy(np.asarray(keys, np.float32), layout)
    am = got_a != ref_a
    rm = got_r != ref_r
    if exact:
        assert not am.any(), f"{am.sum()} angle-code mismatches"
        assert not rm.any(), f"{rm.sum()} radius-code mismatches"
        return 0, 0
    if am.any():
        # a radius tie can also flip the canonical angle; those are radius ties
        ok = po.classify_angle_mismatch(x[am], y[am], m) | rm[am]
        assert ok.all(), f"{(~ok).sum()} non-tie angle mismatches of {am.sum()}"
    if rm.any():
        s32 = np.broadcast_to(s16.astype(np.float32), x.shape)
        ok = po.radius_tie(x[rm], y[rm], s32[rm])
        assert ok.all(), f"{(~ok).sum()} non-tie radius mismatches of {rm.sum()}"
    assert am.mean() <= 1e-5 and rm.mean() <= 1e-5, (am.mean(), rm.mean())
    return int(am.sum()), int(rm.sum())


def peak_close(got, ref, rel: float):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    peak = max(1.0, float(np.abs(ref).max())) if ref.size else 1.0
    err = float(np.abs(got - ref).max()) if ref.size else 0.0
    assert err <= rel * peak, f"max|err| {err:.3e} > {rel:g} * peak {peak:.3e}"
    return err / peak
