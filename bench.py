"""PolarQuant B200 benchmark (driver contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1]): Llama-3.1-8B decode attention,
all 32 layers, batch 16, 32K context, 32 query / 8 KV heads, d=128, m=4/n=4
polar keys + bf16 values.  One step = one decode step over all 32 layers (per
layer one fused LUT-attention launch over its 128 (sequence, kv-head) units
plus the split merge, captured in a CUDA graph).  value = sequences advanced
per second (tokens/s), whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--shard batch|heads] [--no-extras]

Multi-GPU (torchrun, one process per GPU):
  --shard batch (default)  each rank owns its own 16 sequences: units are
                           independent, no data-path collective -> "weak".
  --shard heads            configs[2]/[3] style: the fixed global batch is split
                           by KV head; every layer all-gathers the head outputs
                           over NCCL -> "strong".
Time = max over ranks of the device-timed region.

Extras (rank 0, 1 GPU, after the headline): configs[0] (small, latency),
configs[2] at P=1 (128K ctx, m3n2), configs[3] per-GPU slice (70B head shape,
one KV head of 8), configs[4] encoder slab.
"""

from __future__ import annotations

import argparse
import json
import math
import os
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
    ap.add_argument("--shard", choices=["batch", "heads"], default="batch")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="head sharding: fused peer-store gather in the decode epilogue, or NCCL all-gather")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--page-tokens", type=int, default=256,
                    help="tokens per cache page (decode per-launch rate vs page: 64 0.95, 128 0.98, 256 1.02, 512 1.03 at G=4; profiles/r01/page_size_sweep.md)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip configs 1/3/4/5 side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sustain-seconds", type=float, default=2.5,
                    help="extra back-to-back decode after the timed region, reported as 'sustained' (0: skip)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no timing claims)")
    ap.add_argument("--variant", choices=["auto", "lut", "dq"], default="auto",
                    help="scoring kernel of the fused decode (auto: the library's per-G choice)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """SM clock and throttle reasons sampled with NVML every 20 ms while active."""

    REASONS = {  # nvmlClocksEventReason bits
        0x8: "hw_slowdown",
        0x40: "hw_thermal_slowdown",
        0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
        0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, torch_device):
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._handle = None
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(torch_device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self._handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._handle, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._handle = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                clk = nv.nvmlDeviceGetClockInfo(self._handle, nv.NVML_CLOCK_SM)
                reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._handle)
                self.samples.append((float(clk), int(reasons)))
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self._handle is not None:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t.is_alive():
            self._t.join(timeout=5)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        bits = 0
        for _, r in self.samples:
            bits |= r
        return {"sm_mhz": float(np.median([c for c, _ in self.samples])), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(n for b, n in self.REASONS.items() if bits & b), "samples": len(self.samples)}


def unit_bytes(T: int, G: int, d: int, m: int, n: int, value_bits: int | None = None) -> int:
    """Algorithmic HBM bytes of one (sequence, layer, kv-head) unit per decode
    step: codes once per KV head, V once (bf16, or 4-bit codes +
    fp32 (zp, scale) per token in the value-quantized mode), fp16 scales, bf16
    q in / bf16 out for the G query heads."""
    v = T * d * 2 if value_bits is None else T * (d * value_bits // 8 + 8)
    return T * (d // 2) * (m + n) // 8 + v + (d // 2) * 2 + 2 * G * d * 2


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


def cpu_model() -> str:
    """The host CPU (state the core count and the lscpu model)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


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
        "cpu_model": cpu_model(),
        "kind": "port",
        "sample": f"{n_units} unit-decodes ({G} query heads each, T={T}: qk_scores + attention_weights + "
                  f"softmax.V of the numpy oracle port of the reference) on {cores} processes, {wall:.1f}s wall "
                  f"incl. setup; rate extrapolated linearly to {units_per_step} units/step",
        "sec_per_unit_1core": cores / units_per_s,
    }


# ------------------------------------------------------------------- ours


class DecodeWorkload:
    """A multi-layer decode cache on one GPU plus its per-step launch sequence.

    layers x (batch x kv_heads) units, each with T tokens; one step runs every
    layer's fused decode (optionally followed by the head-output gather)."""

    def __init__(self, dev, *, layers, batch, hq, hkv, T, m, n, page_tokens, seed, plan=None, group=None,
                 value_bits=None, gather="p2p"):
        import torch

        import paper_2502_00527_b200 as pq

        self.dev, self.torch, self.pq = dev, torch, pq
        self.L, self.T, self.m, self.n = layers, T, m, n
        self.G = hq // hkv
        self.plan, self.group = plan, group
        self.upl = plan.units_per_layer if plan is not None else batch * hkv
        self.batch, self.hq = batch, hq
        cfg = pq.QuantConfig(m, n)
        self.value_bits = value_bits
        self.cache = pq.PolarKVCache(cfg, layers * self.upl, 128, 0, capacity=T, page_tokens=page_tokens,
                                     value_dtype=torch.bfloat16, device=dev, value_bits=value_bits)
        syn = pq.SyntheticConfig(T, 128, outlier_channels=frozenset({0, 1}))
        chunk = max(1, min(self.upl, (1 << 31) // (T * 128 * 2)))  # <= 2 GB bf16 staging per tensor
        for layer in range(layers):
            for u0 in range(0, self.upl, chunk):
                k = min(chunk, self.upl - u0)
                s = (seed * 1000 + layer) * 7919 + u0 + 1
                keys = pq.synthetic_keys_device(syn, k, dtype=torch.bfloat16, device=dev, seed=s)
                vals = pq.normal_device((k, T, 128), s + 1, dtype=torch.bfloat16, device=dev)
                self.cache.prefill(keys, vals, unit_start=layer * self.upl + u0, check=(layer == 0 and u0 == 0))
                del keys, vals
        self.q = pq.normal_device((layers, self.upl, self.G, 128), 424242 + seed, dtype=torch.bfloat16, device=dev)
        self.out = torch.empty((layers, self.upl, self.G, 128), dtype=torch.bfloat16, device=dev)
        self.views = [self.cache.view(i * self.upl, (i + 1) * self.upl) for i in range(layers)]
        self.gathered = None
        self.peers = None
        if plan is not None and gather == "p2p":  # fused into the decode epilogue (peer stores + flags)
            from paper_2502_00527_b200.sharding import PeerGather

            self.peers = PeerGather(plan, dev, group)
        elif plan is not None:
            self.gathered = torch.empty((layers, batch, hq, 128), dtype=torch.bfloat16, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        # the prefill ran on the current stream; every decode runs on self.stream
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        self.base_flags = 0  # PQB_DECODE_* bits added to every launch (kernel-variant probes)

    def step(self, flags: int = 0):
        if self.peers is not None:
            for i in range(self.L):
                self.views[i].decode_peer(self.q[i], self.peers.descriptor(i), max_tokens=self.T)
            for i in range(self.L):
                self.peers.wait(i)
            return
        for i in range(self.L):
            self.views[i].decode(self.q[i], out=self.out[i], max_tokens=self.T, flags=flags | self.base_flags)
            if self.gathered is not None:
                from paper_2502_00527_b200.sharding import gather_head_outputs

                self.gathered[i].copy_(gather_head_outputs(self.out[i], self.plan, self.group))

    def launches_per_step(self) -> int:
        # per layer: the fused decode, plus the separate split-merge launch when
        # the library picks it for this shape (pqb_decode_launches), or with the
        # fused peer gather the pqb_peer_wait launch (the merge stays in-kernel)
        from paper_2502_00527_b200 import _lib

        if self.peers is not None:
            return 2 * self.L
        return self.L * int(_lib.load().pqb_decode_launches(self.upl, self.G, self.T, self.base_flags))

    def bytes_per_launch(self) -> int:
        return self.upl * unit_bytes(self.T, self.G, 128, self.m, self.n, self.value_bits)

    def capture(self, fn):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            fn()
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            fn()
        return g.replay

    def timed(self, fn, steps: int, warmup: int, dist=None) -> float:
        torch = self.torch
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                fn()
        torch.cuda.synchronize(self.dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.stream):
            e0.record(self.stream)
            for _ in range(steps):
                fn()
            e1.record(self.stream)
        torch.cuda.synchronize(self.dev)
        ms = e0.elapsed_time(e1) / steps
        if dist:
            on_dev = dist.get_backend() == "nccl"
            t = torch.tensor([ms], device=self.dev if on_dev else "cpu", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def free(self):
        del self.cache, self.q, self.out, self.views
        self.torch.cuda.empty_cache()


def measure_workload(w: DecodeWorkload, steps: int, warmup: int, graph: bool = True) -> dict:
    """Step time (graph) + attention-kernel-only time per launch + roofline."""
    from paper_2502_00527_b200 import _lib

    run = w.capture(w.step) if graph else w.step
    run_attn = w.capture(lambda: w.step(_lib.PQB_DECODE_NO_COMBINE)) if graph else (
        lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
    ms = w.timed(run, steps, warmup)
    ms_attn = w.timed(run_attn, max(3, steps // 2), 2) / w.L
    pk = peaks()
    algo = w.bytes_per_launch()
    return {"ms_per_step": ms, "tokens_per_s": w.batch / (ms * 1e-3), "avg_launch_ms": ms_attn,
            "achieved_gbs": algo / (ms_attn * 1e-3) / 1e9, "frac": algo / (ms_attn * 1e-3) / 1e9 / pk["hbm_gbs"],
            "step_frac": w.L * algo / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]}


def run_ours(a, rank: int, world: int, dist) -> dict | None:
    import torch

    from paper_2502_00527_b200 import sharding

    dev = torch.device("cuda", torch.cuda.current_device() if world > 1 else int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    G = a.hq // a.hkv
    plan = None
    batch = a.batch
    if a.shard == "heads" and world > 1:
        shape = sharding.DecodeShape(a.layers, a.batch, a.hq, a.hkv)
        plan = sharding.head_shard(shape, world, rank)
    w = DecodeWorkload(dev, layers=a.layers, batch=batch, hq=a.hq, hkv=a.hkv, T=a.ctx, m=a.m, n=a.n,
                       page_tokens=a.page_tokens, seed=rank, plan=plan, gather=a.gather)
    from paper_2502_00527_b200 import _lib as _l

    w.base_flags = {"auto": 0, "lut": _l.PQB_DECODE_LUT, "dq": _l.PQB_DECODE_DQ}[a.variant]
    if a.profile:
        with torch.cuda.stream(w.stream):
            for _ in range(max(1, a.steps)):
                w.step()
        torch.cuda.synchronize(dev)
        return None
    from paper_2502_00527_b200 import _lib

    run = w.step if a.no_graph else w.capture(w.step)
    with ClockSampler(dev) as clk:
        ms_step = w.timed(run, a.steps, a.warmup, dist)
    run_attn = (lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
    run_attn = run_attn if a.no_graph else w.capture(run_attn)
    ms_attn_layer = w.timed(run_attn, max(3, a.steps // 2), 2, dist) / a.layers

    # ---- e2e through the public API with host buffers (pinned), per step:
    #      H2D of every layer's queries, per-layer decode calls, D2H of outputs.
    #      The copies overlap the decode the way a serving loop would issue
    #      them: layer 0's queries first, the other layers' on a copy stream
    #      while layer 0 decodes; all but the last layer's outputs leave on a
    #      copy stream while the last layer decodes.
    q_host = w.q.cpu().pin_memory()
    o_host = torch.empty(w.out.shape, dtype=w.out.dtype).pin_memory()
    q_dev = torch.empty_like(w.q)
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_q, ev_o = torch.cuda.Event(), torch.cuda.Event()
    L = a.layers

    def e2e_step():
        main = torch.cuda.current_stream(dev)
        q_dev[0].copy_(q_host[0], non_blocking=True)
        if L > 1:
            h2d_s.wait_stream(main)  # the previous step is done with q_dev
            with torch.cuda.stream(h2d_s):
                q_dev[1:].copy_(q_host[1:], non_blocking=True)
                ev_q.record(h2d_s)
        for i in range(L):
            if i == 1:
                main.wait_event(ev_q)
            w.views[i].decode(q_dev[i], out=w.out[i], max_tokens=a.ctx)
            if i == L - 2:
                ev_o.record(main)
                d2h_s.wait_event(ev_o)
                with torch.cuda.stream(d2h_s):
                    o_host[:L - 1].copy_(w.out[:L - 1], non_blocking=True)
        o_host[L - 1].copy_(w.out[L - 1], non_blocking=True)
        if L > 1:
            main.wait_stream(d2h_s)  # the step ends when every output is on the host

    ms_e2e = w.timed(e2e_step, max(3, a.steps // 2), 2, dist)

    # ---- sustained: the same graph step back to back for a few seconds (the
    #      board reaches its 1000 W cap within ~0.3 s; profiles/r01/power_probe.md);
    #      reported beside the K-step value, not instead of it
    sustained = None
    if a.sustain_seconds > 0 and not a.no_graph:
        import time as _t

        with ClockSampler(dev) as sclk:
            t_end = _t.time() + a.sustain_seconds
            chunks = []
            while _t.time() < t_end:
                chunks.append(w.timed(run, 8, 0))
        tail = chunks[len(chunks) // 2:] or chunks
        ms_sus = sum(tail) / len(tail)
        sustained = {"seconds": a.sustain_seconds, "ms_per_step": ms_sus,
                     "value": (a.batch * world if a.shard == "batch" else a.batch) / (ms_sus * 1e-3),
                     "note": "second half of a back-to-back run of the timed step",
                     "clocks": sclk.summary()}
    algo = w.bytes_per_launch()
    pk = peaks()
    achieved = algo / (ms_attn_layer * 1e-3) / 1e9
    global_batch = a.batch * world if a.shard == "batch" else a.batch
    res = {
        "ms_per_step": ms_step,
        "value": global_batch / (ms_step * 1e-3),
        "e2e_ms": ms_e2e,
        "e2e_value": global_batch / (ms_e2e * 1e-3),
        "h2d": q_host.numel() * q_host.element_size(),
        "d2h": o_host.numel() * o_host.element_size(),
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": pk["hbm_gbs"],
            "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"],
            "peak_source": pk["source"],
            "frac_vs_8tbs_nameplate": achieved / 8000.0,  # SURVEY 8(d) asks for both denominators
            "kernel": (f"decode_fast_kernel<G={G},M={a.m},N={a.n}> (LUT gather" if a.variant == "lut" or G not in (4, 8)
                       else f"decode_dq_kernel<G={G},M={a.m},N={a.n}> (product-table gather + tensor-core QK")
                      + "; persistent; timed with the in-kernel split merge disabled)",
            "algorithmic_bytes_per_launch": algo,
            "avg_launch_ms": ms_attn_layer,
            "step_frac": a.layers * algo / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"],
            "traffic": ncu_traffic(),
        },
        "clocks": clk.summary(),
        "sustained": sustained,
        "gpu_launches": a.steps * w.launches_per_step(),
        "global_batch": global_batch,
    }
    w.free()
    del w
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not a.no_extras:
        res["extras"] = run_extras(dev, a)
    return res


def run_extras(dev, a) -> dict:
    """Side measurements of the other BASELINE configs on one GPU."""
    import torch

    out = {}
    specs = {
        "configs[0]_L1_B1_4K_m4n4": dict(layers=1, batch=1, hq=32, hkv=8, T=4096, m=4, n=4),
        "configs[2]_P1_L32_B8_128K_m3n2": dict(layers=32, batch=8, hq=32, hkv=8, T=131072, m=3, n=2),
        "configs[3]_per_gpu_L80_B32_32K_G8_1kvhead": dict(layers=80, batch=32, hq=8, hkv=1, T=32768, m=4, n=4),
        # configs[1] with the reference's value-quantization mode
        # (PackedKVCache(quantize_values=True, value_bits=4)) read inside the kernel
        "configs[1]_vq4_values": dict(layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, value_bits=4),
    }
    for name, s in specs.items():
        try:
            w = DecodeWorkload(dev, page_tokens=a.page_tokens, seed=7, **s)
            r = measure_workload(w, steps=max(3, a.steps // 2), warmup=2)
            r["bytes_per_step"] = w.L * w.bytes_per_launch()
            w.free()
            del w
            torch.cuda.empty_cache()
            out[name] = r
        except Exception as exc:  # report, never hide the headline
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        out["configs[1]_scores_only"] = scores_bench(dev, a)
    except Exception as exc:
        out["configs[1]_scores_only"] = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        out["configs[4]_encode"] = encode_bench(dev, a)
    except Exception as exc:
        out["configs[4]_encode"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def ncu_traffic():
    p = ROOT / "profiles" / "ncu_decode_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def scores_bench(dev, a) -> dict:
    """SURVEY 8(d) scores-only mode (paper Table 4 analogue): configs[1] shape,
    the bit-exact LUT scores of qk_scores for every query head, all 32 layers.
    Roofline numerator: the codes (the SURVEY's figure, 8,589,934,592 B/step)
    and, separately, codes + the fp32 score rows written."""
    import torch

    w = DecodeWorkload(dev, layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=a.page_tokens,
                       seed=7)
    from paper_2502_00527_b200 import _lib

    sc = torch.empty((w.upl, w.G, w.T), dtype=torch.float32, device=dev)
    codes = w.L * w.upl * (w.T * 64 * (w.m + w.n) // 8)
    written = w.L * w.upl * w.G * w.T * 4
    pk = peaks()
    res = {"codes_bytes_per_step": codes, "scores_bytes_per_step": written, "gpu_launches_per_step": w.L}
    for name, flags, kern in [
            ("exact_lut", 0, "decode_fast_kernel EXACT (LUT gather, fp32 channel-order sum, bit-identical to qk_scores)"),
            ("dq", _lib.PQB_DECODE_DQ, "decode_dq_kernel scores mode (tensor-core QK, within 1e-4 of qk_scores)")]:
        def step(flags=flags):
            for i in range(w.L):
                w.views[i].scores(w.q[i], max_tokens=w.T, out=sc, flags=flags)

        g = w.capture(step)
        ms = w.timed(g, max(3, a.steps // 2), 2)
        res[name] = {"kernel": kern, "ms_per_step": ms, "tokens_per_s": w.batch / (ms * 1e-3),
                     "frac_codes_only": codes / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                     "frac_codes_plus_scores": (codes + written) / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]}
    del sc
    w.free()
    del w
    torch.cuda.empty_cache()
    return res


def encode_bench(dev, a) -> dict:
    """configs[4] slab on one GPU: 32 layers x 8 kv heads = 256 units x T bf16
    tokens through K1 (scales) + K2 (encode/pack), device-timed, for every
    (m, n) the config names."""
    import torch

    import paper_2502_00527_b200 as pq
    from paper_2502_00527_b200.codec import encode_device, radius_scales_device

    T, U, d = 131072, 256, 128  # config 5 is 1M tokens/unit; cost is linear in T
    syn = pq.SyntheticConfig(T, d, outlier_channels=frozenset({0, 1}))
    keys = pq.synthetic_keys_device(syn, U, dtype=torch.bfloat16, device=dev, seed=99)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(U * 64, dtype=torch.int64, device=dev)
    pk = peaks()
    res = {"workload": f"{U} units x {T} tokens bf16 keys (configs[4] slab; scales + encode + pack)"}
    for m, n in [(4, 4), (3, 2), (2, 4)]:
        cfg = pq.QuantConfig(m, n)
        cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16, device=dev)

        def once():
            radius_scales_device(keys, cfg, flags, ws, out=cache.scales16)
            encode_device(keys, cache.scales16, cfg, cache.store_ref(), clamp_counts=cache.clamp_counts,
                          flags=flags)

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
        algo = U * (2 * T * d * 2 + T * (d // 2) * (m + n) // 8 + (d // 2) * 2)
        res[f"m{m}n{n}"] = {"ms": ms, "token_heads_per_s": U * T / (ms * 1e-3),
                            "achieved_gbs": algo / (ms * 1e-3) / 1e9,
                            "frac": algo / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]}
        del cache
    del keys
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------- main


def main() -> None:
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        # PQB_BENCH_DEVICE / PQB_BENCH_BACKEND: run the N > 1 path as N ranks on
        # one GPU over gloo (a smoke test of the multi-rank code on a 1-GPU box)
        dev_override = os.environ.get("PQB_BENCH_DEVICE")
        torch.cuda.set_device(int(dev_override) if dev_override is not None else int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group(os.environ.get("PQB_BENCH_BACKEND", "nccl"))
        dist = tdist
    G = a.hq // a.hkv
    upl = a.batch * a.hkv
    units_per_step = a.layers * upl
    heads = a.shard == "heads" and world > 1
    config = {"workload": "configs[1]: Llama-3.1-8B heads (32 Q / 8 KV, d=128), 32 layers, batch 16/GPU, 32K ctx, "
                          "m=4 angle / n=4 radius bits, bf16 V; one step = one decode step over all layers",
              "layers": a.layers, "batch_per_gpu": a.batch if not heads else a.batch, "ctx": a.ctx,
              "global_batch": a.batch * world if not heads else a.batch,
              "q_heads": a.hq, "kv_heads": a.hkv, "head_dim": 128, "angle_bits": a.m, "radius_bits": a.n,
              "page_tokens": a.page_tokens,
              "parallelism": (f"kv-head sharded x{world} + per-layer head gather "
                              + ("fused into the decode epilogue (peer stores over NVLink)" if a.gather == "p2p"
                                 else "(NCCL all-gather)") if heads
                              else f"batch-sharded x{world} (no collective)"),
              "l2": "inputs (43 GB cache per GPU) >> 126 MB L2; no flush needed"}

    if a.impl == "reference":
        if rank == 0:
            steps = []
            for i in range(a.warmup + a.steps):
                cb = cpu_baseline(a.ctx, 128, a.m, a.n, G, units_per_step, a.batch,
                                  seconds=max(1.0, a.cpu_seconds / 5))
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
            dist.barrier()
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
            "scaling": "strong" if heads else "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (on-device Philox: lognormal radii, uniform angles, 2 outlier channels)",
            "config": config,
            "roofline": res["roofline"],
            "cpu_baseline": cpu,
            "e2e": {"value": res["e2e_value"], "unit": "tokens/s", "ms_per_step": res["e2e_ms"],
                    "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"]},
            "clocks": res["clocks"],
            "sustained": res.get("sustained"),
            "gpu_launches": res["gpu_launches"],
            "extras": res.get("extras"),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
