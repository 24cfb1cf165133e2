"""PolarQuant B200 benchmark (driver contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1]): Llama-3.1-8B decode attention,
all 32 layers, batch 16, 32K context, 32 query / 8 KV heads, d=128, m=4/n=4
polar keys + bf16 values.  One step = one decode step over all 32 layers (per
layer one fused LUT-attention launch over its 128 (sequence, kv-head) units,
captured in a CUDA graph).  value = sequences advanced per second.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU (torchrun), each rank owns its own 16
sequences (batch sharding: every unit is independent, no data-path
collective) -> "scaling": "weak", value = total over ranks, time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PolarQuant decode-attn tokens/s, Llama-3.1-8B heads @32K ctx; % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--page-tokens", type=int, default=128)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-encode", action="store_true", help="skip the config-5 encoder sub-benchmark")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no timing claims)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def unit_bytes(T: int, G: int, d: int, m: int, n: int) -> int:
    """Algorithmic HBM bytes of one (sequence, layer, kv-head) unit per decode
    step: codes once per KV head, V once (bf16), fp16 scales,
    bf16 q in / bf16 out for the G query heads."""
    return T * (d // 2) * (m + n) // 8 + T * d * 2 + (d // 2) * 2 + 2 * G * d * 2


# ------------------------------------------------------------- CPU baseline


def _cpu_worker(args):
    """One host core: build one (sequence, kv-head) unit with the reference
    algorithm (numpy oracle port: prefill untimed -- the GPU step does not
    prefill either), then repeat its decode -- G query heads of qk_scores +
    attention_weights + softmax.V -- until ``seconds`` elapse."""
    T, d, m, n, G, seed, seconds = args
    from oracle import polar_oracle as po

    keys = po.synthetic_keys(T, d, seed=seed, outliers=(0, 1))
    rng = np.random.default_rng([seed, 1])
    vals = rng.standard_normal((T, d)).astype(np.float32)
    q = rng.standard_normal((G, d)).astype(np.float32)
    oc = po.OracleCache(m, n, po.HALF_SPLIT, 0)
    oc.prefill(keys, vals)
    done, t0 = 0, time.perf_counter()
    while True:
        for g in range(G):
            oc.attention(q[g], 1.0 / math.sqrt(d))
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return done, el


def cpu_baseline(T, d, m, n, G, units_per_step, batch, seconds: float) -> dict:
    """Reference CPU path on every host core (one process per core) for
    ~``seconds`` of decode work each, extrapolated linearly to a full step."""
    from concurrent.futures import ProcessPoolExecutor

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=cores) as ex:
        res = list(ex.map(_cpu_worker, [(T, d, m, n, G, 10_001 + i, seconds) for i in range(cores)]))
    wall = time.perf_counter() - t0
    units_per_s = sum(k / el for k, el in res)
    step_s = units_per_step / units_per_s
    n_units = sum(k for k, _ in res)
    return {
        "value": batch / step_s,
        "unit": "tokens/s",
        "cores": cores,
        "kind": "port",
        "sample": f"{n_units} unit-decodes ({G} query heads each, T={T}: qk_scores + attention_weights + "
                  f"softmax.V of the numpy oracle port of the reference) on {cores} processes, {wall:.1f}s wall "
                  f"incl. setup; rate extrapolated linearly to {units_per_step} units/step",
        "sec_per_unit_1core": cores / units_per_s,
    }


# ------------------------------------------------------------------- ours


def run_ours(a, rank: int, world: int, dist) -> dict | None:
    import torch

    import paper_2502_00527_b200 as pq
    from paper_2502_00527_b200 import _lib

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    L, B, Hq, Hkv, T, d = a.layers, a.batch, a.hq, a.hkv, a.ctx, 128
    G = Hq // Hkv
    upl = B * Hkv  # units per layer
    U = L * upl
    cfg = pq.QuantConfig(a.m, a.n)
    cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T, page_tokens=a.page_tokens, value_dtype=torch.bfloat16,
                            device=dev)
    syn = pq.SyntheticConfig(T, d, outlier_channels=frozenset({0, 1}))
    for layer in range(L):  # fill layer by layer (keeps the bf16 staging at 2 GB)
        seed = (rank * 1000 + layer) * 7919 + 1
        keys = pq.synthetic_keys_device(syn, upl, dtype=torch.bfloat16, device=dev, seed=seed)
        vals = pq.normal_device((upl, T, d), seed + 1, dtype=torch.bfloat16, device=dev)
        cache.prefill(keys, vals, unit_start=layer * upl, check=(layer == 0))
        del keys, vals
    q_all = pq.normal_device((L, upl, G, d), 424242 + rank, dtype=torch.bfloat16, device=dev)
    out_all = torch.empty((L, upl, G, d), dtype=torch.bfloat16, device=dev)
    views = [cache.view(layer * upl, (layer + 1) * upl) for layer in range(L)]
    stream = torch.cuda.Stream(device=dev)

    def step():
        for layer in range(L):
            views[layer].decode(q_all[layer], out=out_all[layer], max_tokens=T)

    def attn_only():
        for layer in range(L):
            views[layer].decode(q_all[layer], out=out_all[layer], max_tokens=T, flags=_lib.PQB_DECODE_NO_COMBINE)

    with torch.cuda.stream(stream):
        step()
        attn_only()
    torch.cuda.synchronize(dev)
    splits = _lib.load().pqb_decode_splits(upl, T)
    launches_per_step = L * (2 if splits > 1 else 1)
    graph = None
    if not a.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        graph_attn = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_attn, stream=stream):
            attn_only()
    run = graph.replay if graph else step
    run_attn = graph_attn.replay if graph else attn_only

    if a.profile:
        with torch.cuda.stream(stream):
            for _ in range(max(1, a.steps)):
                step()
        torch.cuda.synchronize(dev)
        return None

    def timed(fn, steps: int, warmup: int) -> float:
        with torch.cuda.stream(stream):
            for _ in range(warmup):
                fn()
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        if dist:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    with ClockSampler(dev.index) as clk:
        ms_step = timed(run, a.steps, a.warmup)
    ms_attn_layer = timed(run_attn, max(3, a.steps // 2), 2) / L

    # ---- e2e through the public API with host buffers (pinned), per step:
    #      H2D of every layer's queries, 32 decode_attention calls, D2H of outputs.
    q_host = q_all.cpu().pin_memory()
    o_host = torch.empty(out_all.shape, dtype=out_all.dtype).pin_memory()
    q_dev = torch.empty_like(q_all)

    def e2e_step_api():
        q_dev.copy_(q_host, non_blocking=True)
        for layer in range(L):
            views[layer].decode(q_dev[layer], out=out_all[layer], max_tokens=T)
        o_host.copy_(out_all, non_blocking=True)

    ms_e2e = timed(e2e_step_api, max(3, a.steps // 2), 2)

    # ---- config-5 style encoder sub-benchmark (bulk prefill, bf16 keys)
    enc = None
    if not a.no_encode:
        enc = encode_bench(dev, rank, a)

    algo = upl * unit_bytes(T, G, d, a.m, a.n)  # per layer launch
    pk = peaks()
    achieved = algo / (ms_attn_layer * 1e-3) / 1e9
    step_bytes = L * algo
    return {
        "ms_per_step": ms_step,
        "value": B * world / (ms_step * 1e-3),
        "e2e_ms": ms_e2e,
        "e2e_value": B * world / (ms_e2e * 1e-3),
        "h2d": q_host.numel() * q_host.element_size(),
        "d2h": o_host.numel() * o_host.element_size(),
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": pk["hbm_gbs"],
            "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"],
            "peak_source": pk["source"],
            "kernel": f"decode_fast_kernel<G={G},M={a.m},N={a.n}> (split partials, no combine)",
            "algorithmic_bytes_per_launch": algo,
            "avg_launch_ms": ms_attn_layer,
            "step_frac": step_bytes / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"],
            "traffic": ncu_traffic(),
        },
        "clocks": clk.summary(),
        "gpu_launches": a.steps * launches_per_step,
        "splits": splits,
        "encode": enc,
    }


def ncu_traffic():
    p = ROOT / "profiles" / "ncu_decode_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def encode_bench(dev, rank: int, a) -> dict:
    """Config 5 sample on one GPU: 32 layers x 8 kv heads x T tokens of bf16
    keys through K1 (scales) + K2 (encode/pack), timed end to end on device."""
    import torch

    import paper_2502_00527_b200 as pq

    T = 131072  # tokens per unit in the timed slab (config 5 is 1M; per-unit work is linear in T)
    U = 256
    d = 128
    syn = pq.SyntheticConfig(T, d, outlier_channels=frozenset({0, 1}))
    keys = pq.synthetic_keys_device(syn, U, dtype=torch.bfloat16, device=dev, seed=99 + rank)
    cfg = pq.QuantConfig(4, 4)
    cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(U * 64, dtype=torch.int64, device=dev)
    from paper_2502_00527_b200.codec import encode_device, radius_scales_device

    def once():
        radius_scales_device(keys, cfg, flags, ws, out=cache.scales16)
        encode_device(keys, cache.scales16, cfg, cache.store_ref(), clamp_counts=cache.clamp_counts, flags=flags)

    for _ in range(2):
        once()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    algo = U * (2 * T * d * 2 + T * (d // 2) * 8 // 8 + (d // 2) * 2)
    pk = peaks()
    del keys, cache
    torch.cuda.empty_cache()
    return {"workload": f"encode {U} units x {T} tokens bf16 (config-5 slab), m4n4", "ms": ms,
            "token_heads_per_s": U * T / (ms * 1e-3), "achieved_gbs": algo / (ms * 1e-3) / 1e9,
            "frac": algo / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]}


# ------------------------------------------------------------------- main


def main() -> None:
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    G = a.hq // a.hkv
    upl = a.batch * a.hkv
    units_per_step = a.layers * upl
    config = {"workload": "configs[1]: Llama-3.1-8B heads (32 Q / 8 KV, d=128), 32 layers, batch 16/GPU, 32K ctx, "
                          "m=4 angle / n=4 radius bits, bf16 V; one step = one decode step over all layers",
              "layers": a.layers, "batch_per_gpu": a.batch, "global_batch": a.batch * world, "ctx": a.ctx,
              "q_heads": a.hq, "kv_heads": a.hkv, "head_dim": 128, "angle_bits": a.m, "radius_bits": a.n,
              "page_tokens": a.page_tokens, "parallelism": f"batch-sharded x{world} (no collective)",
              "l2": "inputs (43 GB cache per GPU) >> 126 MB L2; no flush needed"}

    if a.impl == "reference":
        if rank == 0:
            steps = []
            for i in range(a.warmup + a.steps):
                cb = cpu_baseline(a.ctx, 128, a.m, a.n, G, units_per_step, a.batch, seconds=max(2.0, a.cpu_seconds / 4))
                if i >= a.warmup:
                    steps.append(cb)
            v = float(np.mean([s["value"] for s in steps]))
            line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": a.steps,
                    "warmup": a.warmup, "ms_per_step": a.batch / v * 1e3, "higher_is_better": True,
                    "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                    "impl": "reference",
                    "cpu_baseline": {**steps[-1], "value": v},
                    "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        if dist:
            dist.destroy_process_group()
        return

    res = run_ours(a, rank, world, dist)
    if res is None:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(a.ctx, 128, a.m, a.n, G, units_per_step, a.batch, a.cpu_seconds)
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": res["value"],
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": res["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (on-device Philox: lognormal radii, uniform angles, 2 outlier channels)",
            "config": config,
            "roofline": res["roofline"],
            "cpu_baseline": cpu,
            "e2e": {"value": res["e2e_value"], "unit": "tokens/s", "ms_per_step": res["e2e_ms"],
                    "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"]},
            "clocks": res["clocks"],
            "gpu_launches": res["gpu_launches"],
            "decode_splits": res["splits"],
            "encode": res["encode"],
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
