#!/usr/bin/env python
"""Benchmark of the Inf-MLLM streaming decode + score + evict hot path on B200.

Default workload (BASELINE.json config 1, Llama-2-7B-shaped decode): 32 layers
x 32 heads x head_dim 128, bf16, 8 independent streams per GPU, KV budget 2048
= 1024 recent + 1024 relevant, relevance window W = 32 queries, attention bias
b = 0.01, eviction every E = 128 tokens.  Synthetic q/k/v ~ N(0,1) with 1% of
keys x4 (random-init stand-in; no model weights or datasets).

One bench "step" = one eviction period at steady state: E decode tokens for
every stream through all layers (append + attention + relevance row) followed
by one eviction of every (stream, layer) (score + bias + top-k + in-place
compaction).  value = decode tokens/s of the whole job.

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path (config 1)
  python bench.py --workload cfg3|cfg4 [--budget B]           # configs 3 / 4
  python bench.py --impl reference [...]                      # CPU reference arm
Under torchrun every rank runs its own streams (configs 1 and 4: weak / even
stream partition, no collective on the hot path) or its own KV heads of the
single stream (config 3: one all-reduce of the window scores per eviction).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/sec per stream-batch & \u00b5s/step (attn+score+evict); HBM GB/s vs peak"

WORKLOADS = {
    "cfg0": dict(layers=1, heads_q=8, heads_kv=8, head_dim=64, streams=1, recent=128, relevant=128, window=32,
                 bias=0.01, period=64, spike_prob=4 / 4096, spike_gain=6.0, shard="streams", scaling="weak",
                 dtype="f32",
                 desc="cfg0: CPU-runnable toy, 1L x 8H x 64, fp32, batch 1, budget 128+128, W=32, b=0.01, E=64 "
                      "(L2-resident, launch-bound: the parity config, reported in us/step)"),
    "cfg1": dict(layers=32, heads_q=32, heads_kv=32, head_dim=128, streams=8, recent=1024, relevant=1024, window=32,
                 bias=0.01, period=128, spike_prob=0.01, spike_gain=4.0, shard="streams", scaling="weak",
                 desc="cfg1: Llama-2-7B-shaped decode, 32L x 32H x 128, bf16, 8 streams/GPU, budget 1024+1024, "
                      "W=32, b=0.01, E=128"),
    "cfg3": dict(layers=32, heads_q=32, heads_kv=8, head_dim=128, streams=1, recent=2048, relevant=2048, window=32,
                 bias=0.01, period=256, spike_prob=0.005, spike_gain=4.0, shard="heads", scaling="strong",
                 desc="cfg3: Llama-3-8B GQA-shaped decode, 32L x 32q/8kv x 128, bf16, batch 1, budget 2048+2048, "
                      "W=32, b=0.01, E=256, KV heads sharded over GPUs"),
    "cfg2": dict(layers=32, heads_q=32, heads_kv=32, head_dim=128, streams=4, recent=2048, relevant=2048, window=32,
                 bias=0.01, period=608, image=576, text=32, shard="streams", scaling="weak",
                 desc="cfg2: Vicuna-7B-shaped video stream, 32L x 32H x 128, bf16, 4 streams/GPU, budget 2048+2048, "
                      "frames of 576 image tokens (one tcgen05 prefill chunk) + 32 text tokens, eviction after "
                      "each chunk"),
    "cfg4": dict(layers=32, heads_q=32, heads_kv=32, head_dim=128, streams=256, recent=1024, relevant=1024, window=32,
                 bias=0.01, period=128, spike_prob=0.01, spike_gain=4.0, shard="streams", scaling="strong",
                 desc="cfg4: 256 Llama-2-7B-shaped streams partitioned over GPUs, bf16, W=32, b=0.01, E=128"),
}
CFG = WORKLOADS["cfg1"]


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


NCU_SUMMARY = "profiles/r2_ncu_summary.json"


def _ncu_traffic():
    """DRAM read+write bytes per decode launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, NCU_SUMMARY)) as f:
            return float(json.load(f)["decode_traffic_bytes_per_launch"])
    except Exception:
        return None


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi needs a few hundred ms to its first sample: wait for it,
        # so a timed region shorter than the 200 ms period (config 0) is still
        # bracketed by samples (this one and the one stop() waits for)
        deadline = time.time() + 5.0
        while not self.lines and time.time() < deadline and self.proc.poll() is None:
            time.sleep(0.01)
        self.n0 = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        deadline = time.time() + 0.5  # one sample after the region too
        while len(self.lines) <= getattr(self, "n0", 0) and time.time() < deadline and self.proc.poll() is None:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}




# ------------------------------------------------------------- accounting --
def _elt(c) -> int:
    return 4 if c.get("dtype") == "f32" else 2


def period_bytes(c, hkv: int, moved_rows_per_sl: float) -> dict:
    """Algorithmic HBM bytes of one period, per (stream, layer)."""
    s = _elt(c)
    B, E, D, W, l = c["recent"] + c["relevant"], c["period"], c["head_dim"], c["window"], c["recent"]
    hq = hkv * (c["heads_q"] // c["heads_kv"])
    kv = sum(2 * (B + j) * hkv * D * s for j in range(1, E + 1))
    step_io = E * (hq * D * s + 2 * hkv * D * s + hq * D * 4)
    n_e = B + E
    window = 8 * (n_e - l) * W
    evict = 4 * (n_e - l) + 4 * B + 4 * moved_rows_per_sl * hkv * D * s
    return dict(kv=kv, step_io=step_io, window=window, evict=evict, total=kv + step_io + window + evict)


def decode_launch_bytes(c, hkv: int, n: float, streams: int) -> float:
    """Algorithmic bytes of one decode launch (one layer, all resident streams, cache length n)."""
    s = _elt(c)
    hq = hkv * (c["heads_q"] // c["heads_kv"])
    D = c["head_dim"]
    return streams * (2 * n * hkv * D * s + hq * D * s + 2 * hkv * D * s + hq * D * 4)


def workload_config(c, S, resident, waves, world, job_streams, hq, hkv, use_graph, gathered, sharded,
                    select="layer") -> dict:
    """The `config` object of a bench line (identical keys for both arms)."""
    B, E, L = c["recent"] + c["relevant"], c["period"], c["layers"]
    return {"workload": c["desc"], "streams_per_gpu": S, "resident_streams": resident, "waves": waves,
            "global_streams": job_streams, "layers": L, "heads_q_per_gpu": hq, "heads_kv_per_gpu": hkv,
            "head_dim": c["head_dim"], "budget": B, "window": c["window"], "period": E,
            "step": f"one eviction period: {E} decode tokens x {L} layers x streams + 1 all-layer eviction",
            "l2": ("L2-resident by construction (sub-MB working set, not flushed): launch-bound parity config"
                   if c.get("dtype") == "f32" else
                   "inputs larger than L2 (the whole KV cache is streamed every token)"),
            "graph": (None if use_graph is None else
                      "one CUDA graph per period, per-layer launches" if use_graph else
                      "eager per-token launches (NCCL all-reduce at eviction)"),
            "result_gather": gathered,
            "select": (select if select == "layer" else
                       "kv_head (per KV-head-group decisions: NOT the reference's per-layer selection)"),
            "parallelism": (f"kv-heads sharded x{world}, select=kv_head: no collective" if select == "kv_head" else
                            f"kv-heads sharded x{world} (1 all-reduce of window scores per eviction)"
                            if sharded else f"stream-partitioned x{world}, no hot-path collective")}


def _local_device() -> int:
    return int(os.environ.get("SKV_BENCH_DEVICE", os.environ.get("LOCAL_RANK", 0)))


def _max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------- GPU arm --
def run_gpu(args, rank: int, world: int):
    import torch
    import torch.distributed as dist

    from paper_2409_09086_b200 import EngineConfig, StreamEngine
    from paper_2409_09086_b200.sharding import KvHeadEngine, evict_head_sharded, gather_results, shard_heads

    c = dict(WORKLOADS[args.workload])
    if args.budget:
        c["recent"] = c["relevant"] = args.budget // 2
    L, HQ, HKV, D = c["layers"], c["heads_q"], c["heads_kv"], c["head_dim"]
    l, r, W, E = c["recent"], c["relevant"], c["window"], c["period"]
    B = l + r
    G = HQ // HKV
    dev = torch.device("cuda", _local_device())
    torch.cuda.set_device(dev)
    select = args.select if c["shard"] == "heads" else "layer"
    sharded = c["shard"] == "heads" and world > 1 and select == "layer"
    if c["shard"] == "heads":
        kvs, qsl = shard_heads(HKV, G, world, rank)
        hkv, hq, S = kvs.stop - kvs.start, qsl.stop - qsl.start, c["streams"]
    else:
        hkv, hq = HKV, HQ
        S = c["streams"] if c["scaling"] == "weak" else c["streams"] // world
    # streams resident at once (config 4 at large budgets runs in waves)
    dt = torch.float32 if c.get("dtype") == "f32" else torch.bfloat16
    per_stream = 2 * L * hkv * (B + E) * D * _elt(c) * 1.06
    free = torch.cuda.mem_get_info(dev)[0] - (12 << 30)
    resident = max(1, min(S, int(free // per_stream)))
    waves = -(-S // resident)
    ecfg = EngineConfig(resident, L, hq, hkv, D, l, r, c["bias"], W, B + E, dt,
                        heads_q_total=HQ if c["shard"] == "heads" and select == "layer" else 0)
    eng = KvHeadEngine(ecfg) if select == "kv_head" else StreamEngine(ecfg)
    core = eng.inner if select == "kv_head" else eng  # the StreamEngine holding the device state
    units = hkv if select == "kv_head" else 1          # selection units per stream
    g = torch.Generator(device=dev).manual_seed(1234 + rank)

    def randn(shape):
        return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(dt)

    def spiked_keys(shape_lead):
        k = torch.randn((*shape_lead, hkv, D), generator=g, device=dev, dtype=torch.float32)
        spikes = torch.rand(shape_lead, generator=g, device=dev) < c["spike_prob"]
        k[spikes] *= c["spike_gain"]
        return k.to(dt)

    # steady state: every (stream, layer) holds a full budget of B tokens
    for u in range(resident * units):
        for layer in range(L):
            kf, vf = core.kv_full(u, layer)
            hk = hkv // units
            kk = torch.randn((hk, B, D), generator=g, device=dev)
            kk[:, torch.rand(B, generator=g, device=dev) < c["spike_prob"]] *= c["spike_gain"]
            kf[:, :B] = kk.to(dt)
            vf[:, :B] = randn((hk, B, D))
            core.lib.skv_state_inject(core._h, u, layer, B, None, None, None, 0, None, None)
    # distinct inputs for up to E steps (fewer when many streams are resident), reused cyclically
    T_in = max(1, min(E, int(3e9 // (L * resident * (hq + 2 * hkv) * D * 2))))
    q = randn((T_in, L, resident, hq, D))
    k = spiked_keys((T_in, L, resident))
    v = randn((T_in, L, resident, hkv, D))
    out = torch.empty((L, resident, hq, D), dtype=torch.float32, device=dev)
    kept = torch.full((resident, units, L, B) if units > 1 else (resident, L, B), -1, dtype=torch.int32,
                      device=dev)

    def evict():
        if sharded:
            evict_head_sharded(eng, -1, kept)
        else:
            eng.evict(-1, kept)

    def decode_steps():
        for t in range(E):  # rows are recorded for the last W steps only (run_period's rule)
            eng.decode_step(q[t % T_in], k[t % T_in], v[t % T_in], out, record=t >= E - W)

    def period():
        decode_steps()
        evict()

    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        period()  # reach the steady ring state (and create the NCCL communicator eagerly)
    stream.synchronize()
    launches0 = eng.kernel_launches
    # one CUDA graph per period; head-sharded layer mode captures the NCCL
    # all-reduce of the window scores inside it too, and falls back to eager
    # launches if this NCCL / driver cannot capture it
    # (gloo collectives cannot be captured: eager periods, functional runs only)
    use_graph = not (sharded and dist.get_backend() != "nccl")
    if use_graph:
        try:
            with torch.cuda.stream(stream):
                eng.capture_begin()
                try:
                    period()
                finally:
                    eng.capture_end()
        except Exception as exc:  # noqa: BLE001
            if not sharded:
                raise
            print(f"[bench] NCCL capture failed ({exc}); eager sharded periods", file=sys.stderr)
            torch.cuda.synchronize()
            use_graph = False
    if use_graph:
        launches_per_period = eng.kernel_launches - launches0

        def step():
            eng.replay()
    else:
        with torch.cuda.stream(stream):
            period()
        stream.synchronize()
        launches_per_period = eng.kernel_launches - launches0
        step = period
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    stream.synchronize()

    clocks = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    wave_ms = _max_over_ranks(t0.elapsed_time(t1) / args.steps, world, dev)
    ms = wave_ms * waves  # every resident wave of this rank's streams takes one period

    kc = kept.cpu().numpy()
    mv = core.moved_rows()  # slot map: rows actually moved by the last eviction
    if mv is not None:
        moved = float(mv.mean())
    else:  # dense stable compaction moves every row after the first evicted one
        first_moved = np.argmax(kc != np.arange(B)[None, None, :], axis=-1)
        moved = float(np.mean(B - first_moved))
    pb = period_bytes(c, hkv, moved)
    step_bytes_rank = pb["total"] * resident * L * waves

    # --- dominant kernel (decode + its merge, one launch unit per layer): the
    # eviction is timed with CUDA events on the same stream and removed from the
    # period; the rest is E*L decode launch units.
    with torch.cuda.stream(stream):
        decode_steps()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        evict()
        ev1.record(stream)
    stream.synchronize()
    evict_ms = ev0.elapsed_time(ev1)
    avg_dec_ms = (wave_ms - evict_ms) / (E * L)
    dec_bytes = decode_launch_bytes(c, hkv, B + (E + 1) / 2.0, resident)
    peak, peak_kind = _peaks()
    achieved = dec_bytes / (avg_dec_ms * 1e-3) / 1e9
    span_us = None
    if use_graph and not sharded:  # device timestamps (first CTA start .. last CTA end) of each decode kernel
        core.timing(True)
        with torch.cuda.stream(stream):
            eng.capture_begin()
            period()
            eng.capture_end()
            eng.replay()
        stream.synchronize()
        ts = core.timing_read()[: E * L].astype(np.int64)
        core.timing(False)
        span_us = float(np.mean(ts[:, 1] - ts[:, 0]) / 1e3) if len(ts) else None

    # --- end to end through the public host-buffer API (pinned memory)
    e2e = None
    if args.e2e_steps > 0:
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        oh = torch.empty((L, resident, hq, D), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        steps = E  # one whole eviction period: the engine states (and their cached graphs) repeat

        # shallow engines (config 0): speculative host steps -- each call also
        # launches the next token behind a doorbell gate (skv_host_speculate)
        spec = L <= 2 and not sharded and hasattr(eng, "host_speculation") and not args.no_host_spec
        if spec:
            eng.host_speculation(True, timeout_us=500)

        def host_period():
            for t in range(steps):
                eng.decode_step_host(qh[t % T_in], kh[t % T_in], vh[t % T_in], oh, record=t >= steps - W)
            evict()

        host_period()  # warm-up: one period (captures the per-state host-step graphs)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tic = time.perf_counter()
        host_period()
        torch.cuda.synchronize()
        el = _max_over_ranks(time.perf_counter() - tic, world, dev) * waves
        job_streams = c["streams"] if c["shard"] == "heads" else S * world
        e2e = {
            "value": round(job_streams * steps / el, 2),
            "unit": "tokens/s",
            # a bench step is one period: `steps` tokens, each copying its q/k/v in and its outputs out
            "h2d_bytes_per_step": int(steps * sum(t[0].numel() * t.element_size() for t in (qh, kh, vh))),
            "d2h_bytes_per_step": int(steps * oh.numel() * oh.element_size()),
            "tokens_per_step": steps,
            "host_speculation": bool(spec),
            "note": "one period through skv_decode_step_host (pinned host q/k/v in, f32 outputs out every token -- "
                    "copied, or read / written by the kernels through the mapped pinned buffers where the path "
                    "allows (SKV_HOST_ZC); the layer-group copy pipeline, a per-state CUDA graph or the shallow "
                    "path, as the engine picks; shallow engines: speculative steps, the next token launched behind a "
                    "doorbell gate) + the eviction, wall clock",
        }

    # the one collective outside the hot path: outputs and kept
    # sets of every rank gathered after the timed region
    gathered = None
    if world > 1:
        torch.cuda.synchronize()
        heads_split = c["shard"] == "heads"
        g_out = gather_results(out, dim=2 if heads_split else 1)
        g_kept = kept if sharded else gather_results(kept, dim=1 if heads_split else 0)
        torch.cuda.synchronize()
        gathered = {"op": "all_gather (NCCL) of outputs" + ("" if sharded else " and kept sets"),
                    "bytes": int(g_out.numel() * g_out.element_size() + (0 if sharded else g_kept.numel() * 4)),
                    "timed": False}
    job_streams = c["streams"] if c["shard"] == "heads" else S * world
    value = job_streams * E / (ms * 1e-3)
    step_bytes_job = _max_over_ranks(step_bytes_rank, 1, dev) * world
    res = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "us_per_token_step": round(ms * 1e3 / E, 3),
        "hbm_gbs_step": round(step_bytes_job / world / (ms * 1e-3) / 1e9, 1),
        "hbm_frac_step": round(step_bytes_job / world / (ms * 1e-3) / 1e9 / peak, 4),
        "higher_is_better": True,
        "scaling": c["scaling"],
        "vs_baseline": None,
        "dtype": c.get("dtype", "bf16"),
        "data": "synthetic (seeded N(0,1) q/k/v, key spikes; random cache at budget)",
        "config": workload_config(c, S=S, resident=resident, waves=waves, world=world, job_streams=job_streams,
                                  hq=hq, hkv=hkv, use_graph=use_graph, gathered=gathered, sharded=sharded,
                                  select=select),
        "roofline": {"bound": "hbm", "kernel": _kernel_label(eng.last_decode_kernel, G, c),
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": _ncu_traffic() if args.workload == "cfg1" and not args.budget else None,
                     "traffic_source": NCU_SUMMARY + " (ncu --set full, dram read+write per launch)",
                     "avg_launch_us": round(avg_dec_ms * 1e3, 2), "bytes_per_launch": int(dec_bytes),
                     "evict_ms_per_period": round(evict_ms, 3),
                     "kernel_span_us": round(span_us, 2) if span_us else None,
                     "method": "(timed period - CUDA-event-timed eviction) / (E*L) launches; kernel_span_us = "
                               "device %globaltimer first-CTA-start..last-CTA-end (PDL overlaps neighbours)"},
        "bytes_per_step": {k2: int(v2 * resident * L * waves * world) for k2, v2 in pb.items()},
        "moved_rows_per_eviction": round(moved, 1),
        "gpu_launches": int(launches_per_period * args.steps),
        "clocks": clk,
    }
    if e2e:
        res["e2e"] = e2e
    return res


def _kernel_label(name: str, G: int, c: dict) -> str:
    """The decode kernel the engine ran, as the roofline's `kernel` string."""
    dt = c.get("dtype", "bf16")
    if name == "decode_tc_cluster_kernel":
        return (f"decode_tc_cluster_kernel<{G},mt> (all {c['layers']} layers of a token per launch, one thread-block "
                "cluster per segment; per-layer figures = launch / layers)")
    if name == "decode_tcd_kernel":
        return f"decode_tcd_kernel<{G}> (+ merge_kernel)"
    if name == "decode_tc_kernel":
        return f"decode_tc_kernel<{G},mt> (+ merge_kernel)"
    return f"decode_kernel<{dt},{c['head_dim']},{G}> (+ merge_kernel)"


def run_cfg2(args, rank: int, world: int):
    """Config 2: each step is one video frame per stream -- a 576-token image
    chunk (chunked prefill on the tensor cores) then a 32-token text chunk, all
    32 layers, with an all-layer eviction after each chunk."""
    import torch

    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    c = dict(WORKLOADS["cfg2"])
    L, H, D, S = c["layers"], c["heads_q"], c["head_dim"], c["streams"]
    l, r, W, CI, CT = c["recent"], c["relevant"], c["window"], c["image"], c["text"]
    B = l + r
    dev = torch.device("cuda", _local_device())
    torch.cuda.set_device(dev)
    eng = StreamEngine(EngineConfig(S, L, H, H, D, l, r, c["bias"], W, B + CI + 64, torch.bfloat16))
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    for s in range(S):
        for layer in range(L):
            kf, vf = eng.kv_full(s, layer)
            kf[:, :B] = torch.randn((H, B, D), generator=g, device=dev).to(torch.bfloat16)
            vf[:, :B] = torch.randn((H, B, D), generator=g, device=dev).to(torch.bfloat16)
            eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)

    def chunk_inputs(C, image):
        q = torch.randn((L, S, C, H, D), generator=g, device=dev)
        if image:  # k, v = per-(stream, layer, frame, head, dim) mean + 0.5 N(0, 1)
            k = torch.randn((L, S, 1, H, D), generator=g, device=dev) + 0.5 * torch.randn((L, S, C, H, D), generator=g, device=dev)
            v = torch.randn((L, S, 1, H, D), generator=g, device=dev) + 0.5 * torch.randn((L, S, C, H, D), generator=g, device=dev)
        else:
            k = torch.randn((L, S, C, H, D), generator=g, device=dev)
            v = torch.randn((L, S, C, H, D), generator=g, device=dev)
        return [t.to(torch.bfloat16).contiguous() for t in (q, k, v)]

    qi, ki, vi = chunk_inputs(CI, True)
    qt, kt, vt = chunk_inputs(CT, False)
    oi = torch.empty((S, CI, H, D), dtype=torch.float32, device=dev)
    ot = torch.empty((S, CT, H, D), dtype=torch.float32, device=dev)

    def image_chunk():
        for layer in range(L):
            eng.prefill_chunk(layer, qi[layer], ki[layer], vi[layer], oi, modality=1)

    def frame():
        image_chunk()
        eng.evict(-1)
        for layer in range(L):
            eng.prefill_chunk(layer, qt[layer], kt[layer], vt[layer], ot, modality=0)
        eng.evict(-1)

    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        frame()
        launches0 = eng.kernel_launches
        eng.capture_begin()
        frame()
        eng.capture_end()
        launches_per_frame = eng.kernel_launches - launches0
        for _ in range(args.warmup):
            eng.replay()
    stream.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
        for _ in range(args.steps):
            eng.replay()
        t1.record(stream)
    stream.synchronize()
    clk = clocks.stop()
    ms = _max_over_ranks(t0.elapsed_time(t1) / args.steps, world, dev)  # streams are per rank (weak scaling)
    # the image chunk alone (32 x (append + prefill + row fold)), replayed as its
    # own CUDA graph; and the prefill kernel alone (its average launch, CUDA
    # events on the launching stream) over the same cache state
    import ctypes
    with torch.cuda.stream(stream):
        eng.evict(-1)
    stream.synchronize()
    g_img = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_img, stream=stream):
        image_chunk()
    with torch.cuda.stream(stream):
        eng.evict(-1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g_img.replay()
        e1.record(stream)
        eng.evict(-1)
    stream.synchronize()
    img_ms = e0.elapsed_time(e1)
    # the rest of the frame, phase by phase (eager, CUDA events): eviction
    # after the image chunk, the 32-layer text chunk, the second eviction
    with torch.cuda.stream(stream):
        image_chunk()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        eng.evict(-1)
        ev[1].record(stream)
        for layer in range(L):
            eng.prefill_chunk(layer, qt[layer], kt[layer], vt[layer], ot, modality=0)
        ev[2].record(stream)
        eng.evict(-1)
        ev[3].record(stream)
    stream.synchronize()
    phases = {"image_evict_ms": round(ev[0].elapsed_time(ev[1]), 3),
              "text_chunk_ms": round(ev[1].elapsed_time(ev[2]), 3),
              "text_evict_ms": round(ev[2].elapsed_time(ev[3]), 3)}
    # e2e: the frame through the public API from pinned host buffers -- each
    # layer's chunk q/k/v copied host->device on a copy stream (one layer ahead
    # of the attention that consumes it), the text chunk's last-layer outputs
    # (what the model consumes next) read back to the host every frame
    hin = [t.cpu().pin_memory() for t in (qi, ki, vi, qt, kt, vt)]
    hout = torch.empty(ot.shape, dtype=ot.dtype).pin_memory()
    cps = torch.cuda.Stream(device=dev)
    e2e_frames = max(2, args.steps)

    def frame_host():
        start = torch.cuda.Event()
        start.record(stream)
        cps.wait_event(start)  # the previous frame has consumed its inputs
        for chunk, (hq, hk, hv, dq, dk, dv, dout, mod) in enumerate(
                ((hin[0], hin[1], hin[2], qi, ki, vi, oi, 1), (hin[3], hin[4], hin[5], qt, kt, vt, ot, 0))):
            ready = []
            with torch.cuda.stream(cps):
                for layer in range(L):
                    dq[layer].copy_(hq[layer], non_blocking=True)
                    dk[layer].copy_(hk[layer], non_blocking=True)
                    dv[layer].copy_(hv[layer], non_blocking=True)
                    ev_l = torch.cuda.Event()
                    ev_l.record(cps)
                    ready.append(ev_l)
            with torch.cuda.stream(stream):
                for layer in range(L):
                    stream.wait_event(ready[layer])
                    eng.prefill_chunk(layer, dq[layer], dk[layer], dv[layer], dout, modality=mod)
                eng.evict(-1)
        with torch.cuda.stream(stream):
            hout.copy_(ot, non_blocking=True)

    frame_host()
    stream.synchronize()
    x0 = torch.cuda.Event(enable_timing=True)
    x1 = torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    for _ in range(e2e_frames):
        frame_host()
    x1.record(stream)
    stream.synchronize()
    e2e_ms = _max_over_ranks(x0.elapsed_time(x1) / e2e_frames, world, dev)
    e2e = {"value": round(S * (CI + CT) * world / (e2e_ms * 1e-3), 2), "unit": "tokens/s",
           "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in hin)),
           "d2h_bytes_per_step": int(hout.numel() * hout.element_size()), "steps": e2e_frames,
           "note": "StreamEngine.prefill_chunk per layer from pinned host q/k/v (copy stream one layer ahead), "
                   "evictions, text chunk's last-layer outputs read back per frame"}
    kv_rows = S * L * H * (B + CI + 64)
    kbase, vbase = eng.kv_full(0, 0)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    sh = ctypes.c_void_p(stream.cuda_stream)
    reps = 3
    with torch.cuda.stream(stream):
        for it in range(reps + 1):
            if it == 1:
                k0 = torch.cuda.Event(enable_timing=True)
                k1 = torch.cuda.Event(enable_timing=True)
                k0.record(stream)
            for layer in range(L):
                eng.lib.skv_prefill_attend(P(qi[layer]), S, CI, H, H, P(kbase), P(vbase), L, layer, B + CI + 64, B,
                                           P(oi), 0, None, 0, None, sh)
        k1.record(stream)
    stream.synchronize()
    kern_us = k0.elapsed_time(k1) * 1e3 / (reps * L)
    n0 = B  # every chunk starts from the evicted budget
    flops = 4 * D * (CI * n0 + CI * (CI + 1) / 2) * S * L * H  # useful QK^T + PV flops of the image chunk
    tflops = flops / L / (kern_us * 1e-6) / 1e12
    # the kernel is timed alone (L launches back to back, ~7 ms): the burst peak
    peak_tf, peak_kind = 1630.4, "fallback burst bf16"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak_tf, peak_kind = float(json.load(f)["bf16_tflops"]), "measured burst bf16 (kernel timed alone)"
    except Exception:
        pass
    tokens = S * (CI + CT) * world
    return {
        "metric": METRIC, "value": round(tokens / (ms * 1e-3), 2), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (frame-mean image k/v, N(0,1) text)",
        "config": {"workload": c["desc"], "streams_per_gpu": S, "budget": B, "window": W,
                   "step": "one frame: 576-token image chunk + 32-token text chunk, 32 layers, 2 evictions",
                   "graph": "one CUDA graph per frame",
                   "l2": "inputs larger than L2 (4 x 32 layers x 4.7K tokens of K/V, 10 GB)",
                   "parallelism": f"stream-partitioned x{world}, no hot-path collective"},
        "roofline": {"bound": "tensor", "kernel": "prefill_kernel (576-query image chunk, one layer, 4 streams x 32 heads)",
                     "achieved": round(tflops, 1), "peak": peak_tf, "peak_kind": peak_kind,
                     "unit": "TFLOP/s", "frac": round(tflops / peak_tf, 4), "traffic": None,
                     "avg_launch_us": round(kern_us, 1), "useful_tflop_per_launch": round(flops / L / 1e12, 4),
                     "image_chunk_ms": round(img_ms, 3), **phases,
                     "image_chunk_tflops": round(flops / (img_ms * 1e-3) / 1e12, 1),
                     "note": "useful causal flops (the kernel issues whole 128x128 tiles); image_chunk_ms = 32 x "
                             "(append + prefill + window-row fold) replayed as one CUDA graph; the other phases "
                             "eager, CUDA events on the launching stream"},
        "gpu_launches": int(launches_per_frame * args.steps),
        "clocks": clk,
        "e2e": e2e,
    }


# --------------------------------------------------------------- CPU arm --

def _cpu_proc(conn, lanes, seed, c):
    """Worker process: holds `lanes` (stream, layer) states of the oracle
    (the reference algorithm restated in NumPy f32, one BLAS thread).  On
    request ("period", E) it runs a whole eviction period on every lane --
    E decode steps (append, attention, head-mean row, window push) and one
    eviction (Algorithm 1 + gather_keep + window remap) -- and returns its own
    elapsed time; ("warm", d) runs d decode steps on one lane (untimed)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle.streamkv_oracle import LayerKV, PolicyConfig, RowWindow, attend_heads, head_mean, saddle_decide, \
        bf16_round

    H, D = c["heads_q"], c["head_dim"]
    l, r, W = c["recent"], c["relevant"], c["window"]
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=c["bias"])
    rng = np.random.default_rng(seed)
    stores, wins = [], []
    for _ in range(lanes):
        st = LayerKV(H, D)
        kb = bf16_round(rng.standard_normal((B, H, D)).astype(np.float32))
        vb = bf16_round(rng.standard_normal((B, H, D)).astype(np.float32))
        for t in range(B):
            st.append(kb[t], vb[t], t)
        stores.append(st)
        wins.append(RowWindow(W))
    scale = np.float32(1.0 / np.sqrt(D))
    pos = B
    conn.send("ready")
    while True:
        req = conn.recv()
        if req is None:
            break
        kind, E = req
        steps = E if kind == "period" else 1
        qs = bf16_round(rng.standard_normal((steps, lanes, H, D)).astype(np.float32))
        ks = bf16_round(rng.standard_normal((steps, lanes, H, D)).astype(np.float32))
        vs = bf16_round(rng.standard_normal((steps, lanes, H, D)).astype(np.float32))
        if kind == "warm":
            st = stores[0]
            probs, _ = attend_heads(st.keys(), st.values(), qs[0, 0], scale)
            conn.send((0.0, 0.0))
            continue
        t0 = time.perf_counter()
        for t in range(E):
            for i in range(lanes):
                st = stores[i]
                st.append(ks[t, i], vs[t, i], pos + t)
                probs, _ = attend_heads(st.keys(), st.values(), qs[t, i], scale)
                wins[i].push(head_mean(probs))
        t1 = time.perf_counter()
        for i in range(lanes):
            dec = saddle_decide(wins[i], stores[i].n, cfg)
            stores[i].gather_keep(dec.kept)
            wins[i].remap(dec.kept)
        t2 = time.perf_counter()
        pos += E
        conn.send((t1 - t0, t2 - t1))


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuReference:
    """The reference algorithm (oracle port: the reference is pure Python, so
    there is nothing to compile) on all host cores: one single-threaded
    process per group of (stream, layer) lanes of the config-1 workload.  A
    sample is one WHOLE eviction period of every lane -- 128 decode tokens x
    32 layers x 8 streams plus the all-layer eviction -- measured, not
    extrapolated; the period time is the slowest process's (they run
    concurrently)."""

    def __init__(self, procs: int = None, seed: int = 0):
        c = dict(CFG)
        self.c = c
        self.S, self.E = c["streams"], c["period"]
        lanes_total = c["streams"] * c["layers"]
        procs = procs or min(os.cpu_count() or 1, lanes_total)
        per = [lanes_total // procs + (1 if i < lanes_total % procs else 0) for i in range(procs)]
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for i, n in enumerate(per):
            if n == 0:
                continue
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_proc, args=(b, n, seed + i, c), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for cn in self.conns:
            assert cn.recv() == "ready"
        self.info = {"procs": len(self.procs), "lanes": lanes_total, "host_cpus": os.cpu_count(),
                     "cpu_model": _cpu_model()}

    def warm(self):
        for cn in self.conns:
            cn.send(("warm", 1))
        for cn in self.conns:
            cn.recv()

    def period(self):
        """Seconds of one whole period (all lanes): (job time, decode part, evict part)."""
        for cn in self.conns:
            cn.send(("period", self.E))
        res = [cn.recv() for cn in self.conns]
        tot = [d + e for d, e in res]
        k = int(np.argmax(tot))
        return tot[k], res[k][0], res[k][1]

    def close(self):
        for cn in self.conns:
            cn.send(None)
        for p in self.procs:
            p.join(timeout=10)


def _cpu_sample_text(info, periods):
    return (f"config 1, {periods} whole eviction period(s): {info['lanes']} (stream, layer) lanes x (128 decode "
            f"tokens + 1 eviction) on {info['procs']} single-thread processes ({info['host_cpus']} host CPUs, "
            f"{info['cpu_model']}); measured, not extrapolated")


def cpu_sample(procs: int = None, seed: int = 0):
    """The GPU arm's cpu_baseline leg: one whole period (~10-30 s of CPU work)."""
    ref = CpuReference(procs, seed)
    try:
        ref.warm()
        sec, _, _ = ref.period()
    finally:
        ref.close()
    return ref.S * ref.E / sec, ref.info


def run_reference(args, rank: int, world: int):
    import torch  # noqa: F401  (keeps the import cost identical across arms)

    if rank != 0:
        return None
    ref = CpuReference(seed=100)
    try:
        for _ in range(args.warmup):  # untimed: one decode step per process (page-in, BLAS warm-up)
            ref.warm()
        per = [ref.period() for _ in range(args.steps)]
    finally:
        ref.close()
    info = ref.info
    secs = np.array([p[0] for p in per])
    value = float(ref.S * ref.E * len(secs) / secs.sum())
    c = dict(CFG)
    return {
        "metric": METRIC, "impl": "reference", "value": round(value, 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(float(secs.mean()) * 1e3, 1),
        "us_per_token_step": round(float(secs.mean()) * 1e6 / ref.E, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (bf16-rounded inputs)",
        "data": "synthetic (seeded N(0,1) q/k/v; random cache at budget)",
        "config": workload_config(c, S=c["streams"], resident=c["streams"], waves=1, world=world,
                                  job_streams=c["streams"] * world, hq=c["heads_q"], hkv=c["heads_kv"],
                                  use_graph=None, gathered=None, sharded=False),
        "timing": {"decode_s_per_period": round(float(np.mean([p[1] for p in per])), 3),
                   "evict_s_per_period": round(float(np.mean([p[2] for p in per])), 3),
                   "warmup": "one decode step per process (untimed)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": info["procs"], "kind": "port",
                         "host_cpus": info["host_cpus"], "cpu_model": info["cpu_model"],
                         "sample": _cpu_sample_text(info, args.steps)},
        "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=128)
    ap.add_argument("--no-host-spec", action="store_true", help="e2e leg without speculative host steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="cfg1", choices=sorted(WORKLOADS))
    ap.add_argument("--budget", type=int, default=0, help="config 4 KV budget sweep (1024/2048/4096/8192)")
    ap.add_argument("--select", default="layer", choices=["layer", "kv_head"],
                    help="config 3: per-layer selection over all heads (reference semantics; one all-reduce per "
                         "eviction when sharded) or per KV-head group (no collective; labelled non-reference)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        import torch
        import torch.distributed as dist

        # SKV_BENCH_BACKEND=gloo + SKV_BENCH_DEVICE=0: functional check of the
        # multi-rank path on one GPU (tests/test_gpu_bench.py; not a measurement)
        backend = os.environ.get("SKV_BENCH_BACKEND") or ("nccl" if args.impl == "ours" else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(_local_device())
        dist.init_process_group(backend=backend)
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    elif args.workload == "cfg2":
        res = run_cfg2(args, rank, world)
    else:
        res = run_gpu(args, rank, world)
        if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "cfg1":
            v, info = cpu_sample(seed=7)
            res["cpu_baseline"] = {
                "value": round(v, 3), "unit": "tokens/s", "cores": info["procs"], "kind": "port",
                "host_cpus": info["host_cpus"], "cpu_model": info["cpu_model"], "sample": _cpu_sample_text(info, 1),
            }
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
