"""PolarQuant B200 benchmark (driver contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1]): Llama-3.1-8B decode attention,
all 32 layers, batch 16, 32K context, 32 query / 8 KV heads, d=128, m=4/n=4
polar keys + bf16 values.  One step = one decode step over all 32 layers (per
layer one fused decode launch over its 128 (sequence, kv-head) units plus the
split merge, captured in a CUDA graph).  value = sequences advanced per second
(tokens/s), whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--shard batch|heads] [--no-extras] [--no-parity]

Multi-GPU: one process per GPU.  Under torchrun the ranks come from the
environment; ``--gpus N`` without WORLD_SIZE re-launches itself under
torch.distributed.run with N ranks (ranks beyond the visible GPUs share them,
over gloo, as a functional check of the N > 1 path).
  --shard batch (default)  each rank owns its own 16 sequences: units are
                           independent, no data-path collective -> "weak".
  --shard heads            configs[2]/[3] style: the fixed global batch is split
                           by KV head; the per-layer head-output gather is fused
                           into the decode epilogue (peer stores) -> "strong".
For N > 1 the line also carries configs[2] (m3n2, 128K, KV-head sharded over
the N ranks) and configs[3] (70B shape, G = 8, KV-head sharded with the fused
gather) measured the same way.  Time = max over ranks of the device-timed region.

Value and e2e are timed interleaved over --reps repetitions (median reported,
spread alongside).  After timing, a parity leg checks sampled units of the
timed caches (every unit of layer 0 plus a random sample) against the oracle:
codes bit-exact vs the correctly rounded C restatement, ties counted vs the
numpy restatement of the reference, outputs vs softmax64 . V (oracle/parity.py;
the oracle is the checker only, never on the timed path).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PolarQuant decode-attn tokens/s, Llama-3.1-8B heads @32K ctx; % HBM roofline"
REF_DIR = ROOT / "baseline" / "_ref"  # the unmodified reference, pip-installed


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3, help="interleaved value / e2e repetitions (median reported)")
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
                    help="tokens per cache page (decode per-launch rate vs page: 64 0.95, 128 0.98, 256 1.02, "
                         "512 1.03 at G=4; profiles/r01/page_size_sweep.md)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other configs' side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-parity", action="store_true", help="skip the parity leg")
    ap.add_argument("--parity-sample", type=int, default=16,
                    help="units checked beyond layer 0 (headline); extras check this many in total")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sustain-seconds", type=float, default=2.5,
                    help="extra back-to-back decode after the timed region, reported as 'sustained' (0: skip)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no timing claims)")
    ap.add_argument("--variant", choices=["auto", "lut", "dq"], default="auto",
                    help="scoring kernel of the fused decode (auto: the library's per-G choice)")
    ap.add_argument("--values", choices=["bf16", "f32", "vq2", "vq4", "vq8"], default="bf16",
                    help="value-cache treatment of the headline workload")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json, copy bandwidth)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


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


def unit_bytes(T: int, G: int, d: int, m: int, n: int, values: str = "bf16") -> int:
    """Algorithmic HBM bytes of one (sequence, layer, kv-head) unit per decode
    step: codes once per KV head, V once (bf16 rows, fp32 rows,
    or b-bit codes + fp32 (zp, scale) per token), fp16 scales, bf16 q in /
    bf16 out for the G query heads."""
    v = {"bf16": T * d * 2, "f32": T * d * 4, "vq2": T * (d // 4 + 8), "vq4": T * (d // 2 + 8),
         "vq8": T * (d + 8)}[values]
    return T * (d // 2) * (m + n) // 8 + v + (d // 2) * 2 + 2 * G * d * 2


def spread(xs) -> dict:
    xs = sorted(float(x) for x in xs)
    return {"median": float(np.median(xs)), "min": xs[0], "max": xs[-1], "n": len(xs)}


# ------------------------------------------------------------- CPU baseline


_CPU_UNIT = None


def _cpu_init(T, d, m, n, G, seed, use_ref):
    """Worker initializer: build one (sequence, kv-head) unit with the
    reference's own PackedKVCache.prefill (untimed -- the GPU step does not
    prefill either)."""
    global _CPU_UNIT
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    rng = np.random.default_rng([seed, 1])
    vals = rng.standard_normal((T, d)).astype(np.float32)
    q = rng.standard_normal((G, d)).astype(np.float32)
    if use_ref:
        sys.path.insert(0, str(REF_DIR))
        import polarquant as ref  # the unmodified reference

        keys = ref.gen_synthetic_keys(ref.SyntheticConfig(T, d, outlier_channels=frozenset({0, 1}), seed=seed)).data
        cache = ref.PackedKVCache(ref.QuantConfig(m, n), 0)
        cache.prefill(keys, vals)
        values = cache.values()

        def decode():
            for g in range(G):  # qk_scores + attention_weights, then the restated softmax . V
                w = ref.attention_weights(ref.qk_scores(q[g], cache), 1.0 / math.sqrt(d))
                _ = w @ values
    else:
        from oracle import polar_oracle as po

        keys = po.synthetic_keys(T, d, seed=seed, outliers=(0, 1))
        oc = po.OracleCache(m, n, po.HALF_SPLIT, 0)
        oc.prefill(keys, vals)

        def decode():
            for g in range(G):
                oc.attention(q[g], 1.0 / math.sqrt(d))
    _CPU_UNIT = decode


def _cpu_run(seconds):
    done, t0 = 0, time.perf_counter()
    while True:
        _CPU_UNIT()
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


class CpuBaseline:
    """The reference CPU path on every host core (one process per core, each
    holding one prefilled unit), timed in bounded samples and extrapolated
    linearly in units (the reference is linear in units and T, README.md:25-27)."""

    def __init__(self, T, d, m, n, G, units_per_step, batch):
        from concurrent.futures import ProcessPoolExecutor

        self.use_ref = (REF_DIR / "polarquant" / "__init__.py").exists()
        self.cores = len(os.sched_getaffinity(0))
        self.T, self.G, self.units_per_step, self.batch = T, G, units_per_step, batch
        self.ex = ProcessPoolExecutor(max_workers=self.cores, initializer=_cpu_init,
                                      initargs=(T, d, m, n, G, 10_001, self.use_ref))

    def sample(self, seconds: float) -> dict:
        t0 = time.perf_counter()
        res = list(self.ex.map(_cpu_run, [seconds] * self.cores))
        wall = time.perf_counter() - t0
        units_per_s = sum(k / el for k, el in res)
        step_s = self.units_per_step / units_per_s
        n_units = sum(k for k, _ in res)
        what = ("the unmodified reference (baseline/_ref: PackedKVCache.prefill untimed, qk_scores + "
                "attention_weights + the restated softmax.V)" if self.use_ref else
                "the numpy oracle port of the reference (baseline/_ref absent)")
        return {
            "value": self.batch / step_s,
            "unit": "tokens/s",
            "cores": self.cores,
            "cpu_model": cpu_model(),
            "kind": "reference" if self.use_ref else "port",
            "sample": f"{n_units} unit-decodes ({self.G} query heads each, T={self.T}) of {what} on "
                      f"{self.cores} processes in {wall:.1f}s wall; the rate is extrapolated linearly to the "
                      f"{self.units_per_step} units of one step",
            "sec_per_unit_1core": self.cores / units_per_s,
        }

    def close(self):
        self.ex.shutdown()


# ------------------------------------------------------------------- ours


class DecodeWorkload:
    """A multi-layer decode cache on one GPU plus its per-step launch sequence.

    layers x (batch x kv_heads) units, each with T tokens; one step runs every
    layer's fused decode (with head sharding, fused with the head-output
    gather).  ``keep`` lists local unit ids whose keys / values are kept (on
    the device, bf16) for the parity leg."""

    def __init__(self, dev, *, layers, batch, hq, hkv, T, m, n, page_tokens, seed, plan=None, group=None,
                 values="bf16", gather="p2p", keep=()):
        import torch

        import paper_2502_00527_b200 as pq

        self.dev, self.torch, self.pq = dev, torch, pq
        self.L, self.T, self.m, self.n = layers, T, m, n
        self.G = hq // hkv
        self.plan, self.group = plan, group
        self.upl = plan.units_per_layer if plan is not None else batch * hkv
        self.batch, self.hq = batch, hq
        self.values = values
        cfg = pq.QuantConfig(m, n)
        self.cache = pq.PolarKVCache(cfg, layers * self.upl, 128, 0, capacity=T, page_tokens=page_tokens,
                                     value_dtype=torch.float32 if values == "f32" else torch.bfloat16, device=dev,
                                     value_bits=int(values[2:]) if values.startswith("vq") else None)
        syn = pq.SyntheticConfig(T, 128, outlier_channels=frozenset({0, 1}))
        chunk = max(1, min(self.upl, (1 << 31) // (T * 128 * 2)))  # <= 2 GB bf16 staging per tensor
        keep = set(int(u) for u in keep)
        self.kept: dict[int, tuple] = {}
        for layer in range(layers):
            for u0 in range(0, self.upl, chunk):
                k = min(chunk, self.upl - u0)
                s = (seed * 1000 + layer) * 7919 + u0 + 1
                keys = pq.synthetic_keys_device(syn, k, dtype=torch.bfloat16, device=dev, seed=s)
                vals = pq.normal_device((k, T, 128), s + 1, dtype=torch.bfloat16, device=dev)
                base = layer * self.upl + u0
                self.cache.prefill(keys, vals, unit_start=base, check=False)
                for j in range(k):
                    if base + j in keep:
                        self.kept[base + j] = (keys[j].clone(), vals[j].clone())
                del keys, vals
        self.cache.check()  # any non-finite key / scale overflow in any chunk raises here
        self.q = pq.normal_device((layers, self.upl, self.G, 128), 424242 + seed, dtype=torch.bfloat16, device=dev)
        self.out = torch.empty((layers, self.upl, self.G, 128), dtype=torch.bfloat16, device=dev)
        self.views = [self.cache.view(i * self.upl, (i + 1) * self.upl) for i in range(layers)]
        self.gathered = None
        self.peers = None
        if plan is not None and gather == "p2p":  # fused into the decode epilogue (peer stores + flags)
            from paper_2502_00527_b200.sharding import PeerGather

            try:
                self.peers = PeerGather(plan, dev, group)
            except RuntimeError as exc:  # no P2P between the ranks' GPUs: the NCCL all-gather instead
                print(f"[bench] {exc}; using the NCCL gather", file=sys.stderr, flush=True)
        if plan is not None and self.peers is None:
            self.gathered = torch.empty((layers, batch, hq, 128), dtype=torch.bfloat16, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        # the prefill ran on the current stream; every decode runs on self.stream
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        self.base_flags = 0  # PQB_DECODE_* bits added to every launch (kernel-variant probes)

    # ---- one step: every layer's decode (+ gather)
    def step(self, flags: int = 0, parity: int | None = None):
        if self.peers is not None:
            par = self.peers.next_step() if parity is None else parity
            for i in range(self.L):
                self.views[i].decode_peer(self.q[i], self.peers.descriptor(i, par), max_tokens=self.T)
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
        vdt = {"bf16": _lib.PQB_BF16, "f32": _lib.PQB_F32, "vq2": _lib.PQB_VQ2, "vq4": _lib.PQB_VQ4,
               "vq8": _lib.PQB_VQ8}[self.values]
        return self.L * int(_lib.load().pqb_decode_launches_ex(self.upl, self.G, self.T, self.base_flags, self.m,
                                                               self.n, vdt))

    def bytes_per_launch(self) -> int:
        return self.upl * unit_bytes(self.T, self.G, 128, self.m, self.n, self.values)

    def capture(self, fn):
        """CUDA graph of fn; with the peer gather two graphs (the gathered
        buffer alternates between steps), replayed alternately."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            fn() if self.peers is None else fn(parity=0)
        torch.cuda.synchronize(self.dev)
        if self.peers is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                fn()
            return g.replay
        graphs = []
        for par in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                fn(parity=par)
            graphs.append(g)
        def replay():  # every step (graph or eager) flips the buffer: the double-buffer contract
            graphs[self.peers.next_step()].replay()

        return replay

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
            ms = max_over_ranks(ms, dist, self.dev)
        return ms

    # ---- end to end through the public API with pinned host buffers
    def e2e_fn(self):
        """Per step: H2D of every layer's queries (layer 0 first, the rest on a
        copy stream while layer 0 decodes), the per-layer public decode calls
        (decode / decode_peer + wait), and D2H of every layer's output on a
        copy stream as soon as the layer is done; the step ends when the last
        output is on the host."""
        torch = self.torch
        dev, L = self.dev, self.L
        q_host = self.q.cpu().pin_memory()
        src = self.peers.out[0] if self.peers is not None else self.out
        o_host = torch.empty(src.shape, dtype=src.dtype).pin_memory()
        q_dev = torch.empty_like(self.q)
        h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_q = torch.cuda.Event()
        ev_l = [torch.cuda.Event() for _ in range(L)]

        def e2e_step():
            main = torch.cuda.current_stream(dev)
            q_dev[0].copy_(q_host[0], non_blocking=True)
            if L > 1:
                h2d_s.wait_stream(main)  # the previous step is done with q_dev
                with torch.cuda.stream(h2d_s):
                    q_dev[1:].copy_(q_host[1:], non_blocking=True)
                    ev_q.record(h2d_s)
            par = self.peers.next_step() if self.peers is not None else None
            for i in range(L):
                if i == 1:
                    main.wait_event(ev_q)
                if self.peers is not None:
                    self.views[i].decode_peer(q_dev[i], self.peers.descriptor(i, par), max_tokens=self.T)
                    self.peers.wait(i)
                    out_i = self.peers.out[par, i]
                else:
                    self.views[i].decode(q_dev[i], out=self.out[i], max_tokens=self.T)
                    out_i = self.out[i]
                ev_l[i].record(main)
                d2h_s.wait_event(ev_l[i])
                with torch.cuda.stream(d2h_s):
                    o_host[i].copy_(out_i, non_blocking=True)
            main.wait_stream(d2h_s)  # consumed before the next step may overwrite (double-buffer contract)

        return e2e_step, q_host.numel() * q_host.element_size(), o_host.numel() * o_host.element_size()

    # ---- parity leg (after timing; oracle/parity.py is the checker)
    def parity_jobs(self, units):
        """check_unit kwargs for local units from the last step's outputs."""
        jobs = []
        par = self.peers.parity if self.peers is not None else None
        for u in units:
            keys, vals = self.kept[u]
            layer, j = divmod(u, self.upl)
            if self.peers is not None:
                p = self.plan
                b, h = p.b0 + j // p.kv_heads, p.h0 + j % p.kv_heads
                out = self.peers.out[par, layer, b, h * self.G:(h + 1) * self.G]
            else:
                out = self.out[layer, j]
            a, r = self.cache.code_arrays(u)
            # 4-bit values: the reference's dequantized rows (values(), bit-identical to
            # quantize_uniform / dequantize_uniform, tests/test_oracle_golden.py)
            v = self.cache.values_f32(u) if self.values.startswith("vq") else vals.float()
            jobs.append(dict(keys=keys.float().cpu().numpy(), s16_gpu=self.cache.scales16[u].cpu().numpy(),
                             angle_gpu=a.cpu().numpy(), radius_gpu=r.cpu().numpy(), m=self.m, n=self.n,
                             q=self.q[layer, j].float().cpu().numpy(), values=v.cpu().numpy(),
                             out=out.float().cpu().numpy(), out_bf16=True))
        return jobs

    def free(self):
        del self.cache, self.q, self.out, self.views, self.kept
        if self.peers is not None:
            self.peers.close()  # collective: every rank frees its workloads in the same order
        self.peers = None
        self.torch.cuda.empty_cache()


def max_over_ranks(x: float, dist, dev) -> float:
    import torch

    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], device=dev if on_dev else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def parity_leg(w: DecodeWorkload, units, run, dist=None) -> dict:
    """One more regular step (graph replay), then the oracle checks of the
    sampled units on host threads; summaries of all ranks merged on rank 0."""
    from oracle import parity

    t0 = time.perf_counter()
    with w.torch.cuda.stream(w.stream):
        run()
    w.torch.cuda.synchronize(w.dev)
    # the host's cores shared by the ranks on this node
    threads = max(1, len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))))
    results = parity.check_many(w.parity_jobs(units), threads=threads)
    summ = parity.summarize(results)
    summ["seconds"] = time.perf_counter() - t0
    if dist:
        allsum = [None] * dist.get_world_size()
        dist.all_gather_object(allsum, summ)
        merged = dict(allsum[0])
        for k in ("units", "codes_checked", "scale_mismatches", "exact_code_mismatches", "numpy_ties",
                  "numpy_angle_ties", "numpy_radius_ties", "non_tie_mismatches"):
            merged[k] = sum(s[k] for s in allsum)
        merged["tie_rate"] = merged["numpy_ties"] / max(1, merged["codes_checked"])
        merged["max_out_rel_err"] = max(s["max_out_rel_err"] for s in allsum)
        merged["out_within_tol"] = all(s["out_within_tol"] for s in allsum)
        merged["ranks"] = len(allsum)
        summ = merged
    summ["passed"] = parity.passed(summ)
    return summ


def sample_units(upl: int, layers: int, extra: int, seed: int, all_layer0: bool = True) -> list[int]:
    rng = np.random.default_rng(seed)
    base = list(range(upl)) if all_layer0 else []
    pool = np.arange(upl if all_layer0 else 0, layers * upl)
    more = rng.choice(pool, size=min(extra, pool.size), replace=False).tolist() if pool.size else []
    return sorted(set(base + [int(u) for u in more]))


def run_ours(a, rank: int, world: int, dist) -> dict | None:
    import torch

    from paper_2502_00527_b200 import _lib, sharding

    dev = torch.device("cuda", torch.cuda.current_device())
    G = a.hq // a.hkv
    plan = None
    batch = a.batch
    if a.shard == "heads" and world > 1:
        shape = sharding.DecodeShape(a.layers, a.batch, a.hq, a.hkv)
        plan = sharding.head_shard(shape, world, rank)
    upl = plan.units_per_layer if plan is not None else a.batch * a.hkv
    # every unit of layer 0 on rank 0; the other ranks a random sample
    keep = ([] if a.no_parity or a.profile
            else sample_units(upl, a.layers, a.parity_sample, 77 + rank, all_layer0=rank == 0))
    w = DecodeWorkload(dev, layers=a.layers, batch=batch, hq=a.hq, hkv=a.hkv, T=a.ctx, m=a.m, n=a.n,
                       page_tokens=a.page_tokens, seed=rank, plan=plan, gather=a.gather, values=a.values,
                       keep=keep, group=None)
    w.base_flags = {"auto": 0, "lut": _lib.PQB_DECODE_LUT, "dq": _lib.PQB_DECODE_DQ}[a.variant]
    if a.profile:
        with torch.cuda.stream(w.stream):
            for _ in range(max(1, a.steps)):
                w.step()
        torch.cuda.synchronize(dev)
        return None

    run = w.step if a.no_graph else w.capture(w.step)
    e2e_step, h2d, d2h = w.e2e_fn()
    ms_v, ms_e = [], []
    with ClockSampler(dev) as clk:
        for rep in range(max(1, a.reps)):  # value and e2e interleaved
            ms_v.append(w.timed(run, a.steps, a.warmup if rep == 0 else 2, dist))
            ms_e.append(w.timed(e2e_step, a.steps, a.warmup if rep == 0 else 2, dist))
    ms_step, ms_e2e = float(np.median(ms_v)), float(np.median(ms_e))

    # kernel-only rate of the dominant launch (roofline): the same step with
    # the split merge skipped (PQB_DECODE_NO_COMBINE) -- the attention kernel's
    # launches alone, stated as such; step_frac (below) includes the merge
    if w.peers is None:
        run_attn = (lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
        run_attn = run_attn if a.no_graph else w.capture(run_attn)
        ms_attn_layer = w.timed(run_attn, max(3, a.steps // 2), 2, dist) / a.layers
    else:
        ms_attn_layer = None

    parity = parity_leg(w, keep, run, dist) if keep else None

    # ---- sustained: the same graph step back to back for a few seconds (the
    #      board reaches its 1000 W cap within ~0.3 s; profiles/r01/power_probe.md)
    sustained = None
    if a.sustain_seconds > 0 and not a.no_graph:
        with ClockSampler(dev) as sclk:
            t_end = time.time() + a.sustain_seconds
            chunks = []
            while time.time() < t_end:
                chunks.append(w.timed(run, 8, 0))
        tail = chunks[len(chunks) // 2:] or chunks
        ms_sus = sum(tail) / len(tail)
        gb = a.batch * world if a.shard == "batch" else a.batch
        sustained = {"seconds": a.sustain_seconds, "ms_per_step": ms_sus, "value": gb / (ms_sus * 1e-3),
                     "note": "second half of a back-to-back run of the timed step", "clocks": sclk.summary()}
    algo = w.bytes_per_launch()
    pk = peaks()
    global_batch = a.batch * world if a.shard == "batch" else a.batch
    step_frac = a.layers * algo / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"]
    kern = (f"decode_fast_kernel<G={G},M={a.m},N={a.n}> (LUT gather)" if a.variant == "lut" or G not in (4, 8)
            else f"decode_dq_kernel<G={G},M={a.m},N={a.n}> (product-table gather + tensor-core QK, "
                 f"{'CUDA-core fp32' if a.values == 'f32' else 'tensor-core'} P.V)")
    if ms_attn_layer is not None:
        achieved = algo / (ms_attn_layer * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"],
                "frac_basis": "attention kernel launches alone: the per-layer launch timed with the split merge "
                              "skipped (PQB_DECODE_NO_COMBINE), CUDA events on the launch stream; step_frac "
                              "includes the merge and every launch of the step"}
    else:
        achieved = a.layers * algo / (ms_step * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "frac_basis": "whole step (fused decode + gather launches)"}
    roof.update({
        "peak_source": pk["source"],
        "frac_vs_8tbs_nameplate": achieved / 8000.0,  # SURVEY 8(d) asks for both denominators
        "kernel": kern,
        "algorithmic_bytes_per_launch": algo,
        "bytes_formula": "per unit T*(d/2)*(m+n)/8 codes + V + (d/2)*2 scales + 2*G*d*2 q/out (SURVEY 8(d))",
        "avg_launch_ms": ms_attn_layer,
        "step_frac": step_frac,
        "traffic": ncu_traffic() if a.values == "bf16" and a.m == 4 and a.n == 4 and G == 4 else None,
    })
    if kern.startswith("decode_dq"):  # 1: the product table at its fixed shared address (the fast build)
        roof["dq_smem_layout"] = {0: "none", 1: "prmt_table", 2: "linear_fallback"}[
            int(_lib.load().pqb_decode_dq_layout())]
    res = {
        "ms_per_step": ms_step,
        "value": global_batch / (ms_step * 1e-3),
        "value_reps": spread(global_batch / (m * 1e-3) for m in ms_v),
        "e2e_ms": ms_e2e,
        "e2e_value": global_batch / (ms_e2e * 1e-3),
        "e2e_reps": spread(global_batch / (m * 1e-3) for m in ms_e),
        "h2d": h2d,
        "d2h": d2h,
        "roofline": roof,
        "clocks": clk.summary(),
        "sustained": sustained,
        "gpu_launches": a.steps * w.launches_per_step(),
        "global_batch": global_batch,
        "parity": parity,
    }
    w.free()
    del w
    torch.cuda.empty_cache()
    if not a.no_extras:
        res["extras"] = run_extras(dev, a, rank, world, dist)
    return res


def measure_workload(w: DecodeWorkload, steps: int, warmup: int, dist=None, graph: bool = True) -> dict:
    """Step time (graph) + attention-kernel-only time per launch + roofline."""
    from paper_2502_00527_b200 import _lib

    run = w.capture(w.step) if graph else w.step
    ms = w.timed(run, steps, warmup, dist)
    pk = peaks()
    algo = w.bytes_per_launch()
    r = {"ms_per_step": ms, "step_frac": w.L * algo / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
         "gpu_launches_per_step": w.launches_per_step()}
    if w.peers is None:
        run_attn = w.capture(lambda: w.step(_lib.PQB_DECODE_NO_COMBINE)) if graph else (
            lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
        ms_attn = w.timed(run_attn, max(3, steps // 2), 2, dist) / w.L
        r.update({"avg_launch_ms": ms_attn, "achieved_gbs": algo / (ms_attn * 1e-3) / 1e9,
                  "frac": algo / (ms_attn * 1e-3) / 1e9 / pk["hbm_gbs"],
                  "frac_basis": "kernel only (split merge skipped)"})
    r["_run"] = run
    return r


def run_extras(dev, a, rank: int, world: int, dist) -> dict:
    """The other BASELINE configs.  N = 1: per-GPU side measurements on rank 0.
    N > 1: configs[2] and configs[3] KV-head sharded over the N ranks with the
    fused head-output gather, timed as the max over ranks."""
    import torch

    from paper_2502_00527_b200 import sharding

    out = {}
    if world == 1:
        specs = {
            "configs[0]_L1_B1_4K_m4n4": dict(layers=1, batch=1, hq=32, hkv=8, T=4096, m=4, n=4),
            "configs[2]_P1_L32_B8_128K_m3n2": dict(layers=32, batch=8, hq=32, hkv=8, T=131072, m=3, n=2),
            "configs[3]_per_gpu_L80_B32_32K_G8_1kvhead": dict(layers=80, batch=32, hq=8, hkv=1, T=32768, m=4, n=4),
            # configs[1] with the reference's value-quantization mode
            # (PackedKVCache(quantize_values=True, value_bits=4)) read inside the kernel
            "configs[1]_vq4_values": dict(layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, values="vq4"),
            "configs[1]_vq2_values": dict(layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, values="vq2"),
            "configs[1]_vq8_values": dict(layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, values="vq8"),
            # the reference's default value cache: full-precision fp32 rows (kv_cache.py:8-9, :209)
            "configs[1]_f32_values": dict(layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, values="f32"),
        }
        parity_of = {"configs[2]_P1_L32_B8_128K_m3n2", "configs[3]_per_gpu_L80_B32_32K_G8_1kvhead",
                     "configs[1]_f32_values", "configs[1]_vq4_values", "configs[1]_vq2_values",
                     "configs[1]_vq8_values"}
        for name, s in specs.items():
            try:
                upl = s["batch"] * s["hkv"]
                keep = (sample_units(upl, s["layers"], max(1, a.parity_sample // 2), 5, all_layer0=False)
                        if name in parity_of and not a.no_parity else [])
                w = DecodeWorkload(dev, page_tokens=a.page_tokens, seed=7, keep=keep, **s)
                r = measure_workload(w, steps=max(3, a.steps // 2), warmup=2)
                r["tokens_per_s"] = s["batch"] / (r["ms_per_step"] * 1e-3)
                r["bytes_per_step"] = w.L * w.bytes_per_launch()
                run = r.pop("_run")
                if keep:
                    r["parity"] = parity_leg(w, keep, run)
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
    # N > 1: the configs whose layers span GPUs (KV-head sharding + fused gather)
    per_gpu_budget = 0.8 * torch.cuda.mem_get_info(dev)[1] / max(1, ranks_per_device(world))
    specs = {
        f"configs[2]_P{world}_L32_B8_128K_m3n2_kvhead_sharded": dict(layers=32, batch=8, hq=32, hkv=8, T=131072,
                                                                      m=3, n=2),
        f"configs[3]_P{world}_L80_B32_32K_G8_kvhead_sharded": dict(layers=80, batch=32, hq=64, hkv=8, T=32768,
                                                                    m=4, n=4),
    }
    for name, s in specs.items():
        try:
            shape = sharding.DecodeShape(s["layers"], s["batch"], s["hq"], s["hkv"])
            plan = sharding.head_shard(shape, world, rank)
            per_unit = unit_bytes(s["T"], s["hq"] // s["hkv"], 128, s["m"], s["n"])
            layers = s["layers"]
            fit = int(per_gpu_budget // (plan.units_per_layer * per_unit))
            if fit < layers:  # more ranks than GPUs: fewer layers, stated in the line
                layers = max(1, fit)
                shape = sharding.DecodeShape(layers, s["batch"], s["hq"], s["hkv"])
                plan = sharding.head_shard(shape, world, rank)
            keep = [] if a.no_parity else sample_units(plan.units_per_layer, layers, 2, 9 + rank, all_layer0=False)
            w = DecodeWorkload(dev, layers=layers, batch=s["batch"], hq=s["hq"], hkv=s["hkv"], T=s["T"], m=s["m"],
                               n=s["n"], page_tokens=a.page_tokens, seed=11 + rank, plan=plan, gather="p2p",
                               keep=keep)
            r = measure_workload(w, steps=max(3, a.steps // 2), warmup=2, dist=dist)
            run = r.pop("_run")
            r["layers"] = layers
            r["tokens_per_s"] = s["batch"] / (r["ms_per_step"] * 1e-3)
            r["tokens_per_s_full_depth"] = s["batch"] / (r["ms_per_step"] * s["layers"] / layers * 1e-3)
            r["scaling"] = "strong (fixed global batch split by KV head)"
            r["bytes_per_step_per_gpu"] = w.L * w.bytes_per_launch()
            if keep:
                r["parity"] = parity_leg(w, keep, run, dist)
            r["gather"] = ("fused into the decode epilogue (peer stores, CUDA IPC)" if w.peers is not None
                           else "NCCL all-gather (no P2P access between the ranks' GPUs)")
            w.free()
            del w
            torch.cuda.empty_cache()
            out[name] = r
        except Exception as exc:
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def ranks_per_device(world: int) -> int:
    import torch

    return max(1, math.ceil(world / max(1, torch.cuda.device_count())))


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
    res = {"workload": f"{U} units x {T} tokens bf16 keys (configs[4] slab; scales + encode + pack)",
           "inputs_vs_l2": "8.6 GB of keys per pass >> 126 MB L2"}
    for m, n in [(4, 4), (3, 2), (2, 4), (2, 2), (3, 4), (4, 2)]:
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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(a) -> None:
    """``--gpus N`` outside torchrun: run this script under torch.distributed.run
    with N ranks (one process per GPU) and exit with its status."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def config_of(a, world: int, heads: bool) -> dict:
    return {"workload": "configs[1]: Llama-3.1-8B heads (32 Q / 8 KV, d=128), 32 layers, batch 16/GPU, 32K ctx, "
                        f"m=4 angle / n=4 radius bits, {a.values} V; one step = one decode step over all layers",
            "layers": a.layers, "batch_per_gpu": a.batch, "ctx": a.ctx,
            "global_batch": a.batch * world if not heads else a.batch,
            "q_heads": a.hq, "kv_heads": a.hkv, "head_dim": 128, "angle_bits": a.m, "radius_bits": a.n,
            "values": a.values, "page_tokens": a.page_tokens,
            "parallelism": (f"kv-head sharded x{world} + per-layer head gather "
                            + ("fused into the decode epilogue (peer stores over NVLink)" if a.gather == "p2p"
                               else "(NCCL all-gather)") if heads
                            else f"batch-sharded x{world} (no collective)"),
            "l2": "inputs (43 GB cache per GPU) >> 126 MB L2; no flush needed"}


def main() -> None:
    a = parse()
    maybe_spawn(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    import torch

    ndev = max(1, torch.cuda.device_count()) if torch.cuda.is_available() else 1
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(int(os.environ.get("PQB_BENCH_DEVICE", local % ndev)))
    if world > 1:
        import torch.distributed as tdist

        # NCCL needs one GPU per rank; with more ranks than GPUs (a functional
        # check on a small box) the host-side reductions run over gloo -- the
        # data path has no collective in either case
        backend = os.environ.get("PQB_BENCH_BACKEND", "nccl" if world <= ndev else "gloo")
        tdist.init_process_group(backend)
        dist = tdist
    G = a.hq // a.hkv
    heads = a.shard == "heads" and world > 1
    config = config_of(a, world, heads)
    units_per_step = a.layers * a.batch * a.hkv

    if a.impl == "reference":
        if rank == 0:
            cb = CpuBaseline(a.ctx, 128, a.m, a.n, G, units_per_step, a.batch)
            steps = []
            per = max(1.0, a.cpu_seconds / 5)
            for i in range(a.warmup + a.steps):
                s = cb.sample(per)
                if i >= a.warmup:
                    steps.append(s)
            cb.close()
            v = float(np.median([s["value"] for s in steps]))
            line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": a.steps,
                    "warmup": a.warmup, "ms_per_step": a.batch / v * 1e3, "higher_is_better": True,
                    "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                    "impl": "reference",
                    "cpu_baseline": {**steps[-1], "value": v,
                                     "step_spread": spread(s["value"] for s in steps)},
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
        cb = CpuBaseline(a.ctx, 128, a.m, a.n, G, units_per_step, a.batch)
        cpu = cb.sample(a.cpu_seconds)
        cb.close()
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
            "dtype": "bf16",
            "dtype_detail": (f"q, out and {a.values} values as stored; {a.m}-bit angle / {a.n}-bit radius key "
                             "codes; scores via fp16 hi+lo tensor-core products with fp32 accumulation; "
                             "online softmax and P.V accumulation in fp32"),
            "data": "synthetic (on-device Philox: lognormal radii, uniform angles, 2 outlier channels; "
                    "N(0,1) values and queries)",
            "config": config,
            "value_reps": res["value_reps"],
            "roofline": res["roofline"],
            "cpu_baseline": cpu,
            "e2e": {"value": res["e2e_value"], "unit": "tokens/s", "ms_per_step": res["e2e_ms"],
                    "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"], "reps": res["e2e_reps"],
                    "path": "public API per layer (UnitView.decode / decode_peer + wait) with pinned host q in "
                            "and outputs out every step, copies overlapped on copy streams"},
            "clocks": res["clocks"],
            "sustained": res.get("sustained"),
            "gpu_launches": res["gpu_launches"],
            "parity": res.get("parity"),
            "extras": res.get("extras"),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
