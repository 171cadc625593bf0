#!/usr/bin/env python
"""Benchmark of the WSVD per-head low-rank decode layer on B200.

Metric (BASELINE.json): decode-attention us/layer and tokens/s at the
LLaVA-1.5-7B attention shape (32 heads x 128, E = 4096), per-head rank 32,
ctx 4K, bf16 storage / fp32 accumulate (configs[1]), with the fraction of the
HBM roofline of the dominant kernel.

One step = one attention-layer decode step for every sequence
(pipe::decode_factored's body, pipeline.cpp:320-329): latent projection of
the new token (Q/K/V for every head), latent-cache append, fused decode
attention over the cache, O-projection; on N > 1 GPUs the heads are sharded
and one NCCL all-reduce sums the O-projection partials.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Scaling is weak: global batch = 16 * N sequences, heads sharded N ways, so
every GPU streams the same 268 MB of latent cache per step.  The line also
carries ``strong_scaling``: north_star config 4 (13B, r48, W4A8, INT8 cache)
at a FIXED global batch of 64 with its 40 heads sharded over the N GPUs.

Steps rotate over ``--layers`` (default 8) independent layers, each with its
own factors, W_o and latent cache, so a step's weights were last read 8 steps
(2.4 GB of traffic) earlier and cannot be served from L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: E, nh, H, r, batch per GPU-equivalent, ctx, cache dtype, weight dtype
    "7b-r32-b16-ctx4k-bf16": dict(E=4096, nh=32, H=128, r=32, B=16, L=4096, cache="bf16",
                                  weights="bf16"),
    "7b-r32-b1-ctx2k-f32": dict(E=4096, nh=32, H=128, r=32, B=1, L=2048, cache="f32",
                                weights="f32"),
    "7b-r32-b32-ctx4k-w8a8-i8cache": dict(E=4096, nh=32, H=128, r=32, B=32, L=4096, cache="i8",
                                          weights="i8"),
    "13b-r48-b64-ctx8k-w4a8-i8cache": dict(E=5120, nh=40, H=128, r=48, B=64, L=8192, cache="i8",
                                           weights="i4"),
}
# config 5: the 32-layer stack; every GPU holds one 8-way head shard (4 heads),
# N GPUs run N of the 8 shards with the O-projection all-reduce among them
STACK_CONFIGS = {
    "7b-stack32-r32-b128-ctx32k-bf16": dict(E=4096, nh=32, H=128, r=32, B=128, L=32768, cache="bf16",
                                            weights="bf16", layers=32, shard_of=8),
}
DEFAULT_CONFIG = "7b-r32-b16-ctx4k-bf16"
METRIC = "WSVD decode attn µs/layer & tokens/s (LLaVA-7B shape, ctx 4K); % HBM roofline"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------ clocks ------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------- synthetic layer --
def synthetic_layer(cfg, seed=0):
    """Random-init factors of the config's shape (decode-bench recipe,
    wsvd_main.cpp:360-391: A ~ N(0, 1/E), B ~ N(0, 1/r)) and W_o ~ N(0, 1/E)
    (toymodel.cpp:81,90).  numpy PCG64 streams; no checkpoint exists offline."""
    from paper_2604_02570_b200.decode import HeadFactors, HeadProjection, LayerFactors, Role
    E, nh, H, r = cfg["E"], cfg["nh"], cfg["H"], cfg["r"]
    rng = np.random.default_rng(seed)
    heads = []
    for h in range(nh):
        roles = []
        for role in range(3):
            a = rng.standard_normal((E, r)) / math.sqrt(E)
            b = rng.standard_normal((r, H)) / math.sqrt(r)
            roles.append(HeadFactors(a=a, b=b, rank=r, head=h, role=Role(role)))
        heads.append(HeadProjection(*roles))
    f = LayerFactors(heads=heads, embed_dim=E, head_dim=H)
    w_o = rng.standard_normal((nh * H, E)) / math.sqrt(E)
    return f, w_o


def l2_statement(NL, attn_bytes, step_bytes, l2_bytes):
    """Whether a step's inputs can be L2-resident: each step reads its layer's
    cache and weights, last touched NL steps earlier; the cycle is compared with
    the device's L2 size (queried)."""
    cycle = NL * step_bytes
    verdict = "inputs larger than L2" if cycle > l2_bytes else "WARNING: the rotating working set fits in L2"
    return (f"{verdict}: L2 {l2_bytes / 1e6:.0f} MB; {NL} rotating layers, each step reads its layer's "
            f"{attn_bytes / 1e6:.0f} MB latent cache and {(step_bytes - attn_bytes) / 1e6:.0f} MB of weights last "
            f"touched {NL} steps earlier ({cycle / 1e9:.2f} GB cycle)")


def algorithmic_bytes(cfg, B, nh_g, L):
    """each byte counted once.  Returns (attention-kernel
    bytes per launch, whole-step bytes)."""
    E, H, r = cfg["E"], cfg["H"], cfg["r"]
    cb = {"f32": 4, "bf16": 2, "i8": 1}[cfg["cache"]]
    wb = {"f32": 4, "bf16": 2, "i8": 1, "i4": 0.5}[cfg["weights"]]
    cache = B * L * nh_g * 2 * r * cb + (B * L * nh_g * 2 * 2 if cfg["cache"] == "i8" else 0)
    bfac = nh_g * 3 * r * H * (2 if wb == 2 else (4 if wb == 4 else 1))
    attn = cache + B * nh_g * r * 4 + nh_g * r * H * (2 if wb == 2 else 4) + B * nh_g * H * 4
    a_w = E * nh_g * 3 * r * wb + (nh_g * 3 * r * 4 if wb < 2 else 0)
    oproj = nh_g * r * E * 2  # W'_o = B_V . W_o (V path folded into the O-projection)
    step = cache + a_w + bfac + B * E * 4 + B * nh_g * 2 * r * cb + B * nh_g * H * 4 + oproj + B * E * 4
    return attn, step


# ------------------------------------------------------------ our arm -----
def run_ours(args, cfg_name, cfg):
    import torch
    import torch.distributed as dist

    from paper_2604_02570_b200 import _native as N
    from paper_2604_02570_b200.layer import DecodeLayer
    from paper_2604_02570_b200.sharding import NcclComm, shard_factors, shard_oproj

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N.lib()
    B = cfg["B"] * world                       # weak scaling: 16 sequences per GPU-equivalent
    nh_g = cfg["nh"] // world
    E, H = cfg["E"], cfg["H"]
    L = cfg["L"]
    W, K = args.warmup, args.steps
    cap = L + W + 2 * K + 120  # timed steps, then the e2e steps (+ their warm-ups), per layer at most

    t0 = time.time()
    # args.layers rotating layers (own factors, W_o and cache each), step i on
    # layer i mod n: the weights of a step were last touched n steps earlier,
    # so neither they nor the cache can be served from the 126 MB L2
    NL = max(1, args.layers)
    layers = []
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + args.seed)
    pre = L - 2 - W  # every layer holds ~L - 1 tokens when the timed steps run
    for li in range(NL):
        f, w_o = synthetic_layer(cfg, seed=args.seed + 7919 * li)
        fs = shard_factors(f, world, rank)
        wo_s = shard_oproj(w_o, cfg["nh"], H, world, rank)
        lay = DecodeLayer(fs, wo_s, batch=B, capacity=cap, cache_dtype=cfg["cache"],
                          weight_dtype=cfg["weights"], oproj_dtype="bf16", device=local,
                          head_offset=rank * nh_g)
        if li == 0:
            # prefill through the projection on the device (untimed setup)
            chunk = 256
            for t0_ in range(0, pre, chunk):
                n = min(chunk, pre - t0_)
                xs = torch.randn((n, B, E), generator=gen, device=dev, dtype=torch.float32)
                lay.prefill(xs)
        else:
            lay.fill_synthetic(pre, seed=li)  # synthetic N(0,1) latents, same length
        layers.append(lay)
    layer = layers[0]
    torch.cuda.synchronize()
    log(f"[rank {rank}] setup {time.time() - t0:.1f}s, {NL} layers, cache length {layer.length()}")

    comm = NcclComm(world, rank, local) if world > 1 else None
    xs = torch.randn((W + K + 2, B, E), generator=gen, device=dev, dtype=torch.float32)
    y = torch.empty((B, E), device=dev, dtype=torch.float32)
    out = torch.empty((B, nh_g, H), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    # Single GPU: the NL layers are a decode chain (layer l + 1's token = layer
    # l's output, pipe::decode_factored's layer loop without the FFN), run as
    # ONE persistent kernel per pass over the layers (wsvd_chain_step); a
    # timed "step" is still one layer step of every sequence.  N > 1: every
    # layer step is its own launch followed by the NCCL all-reduce.
    from paper_2604_02570_b200.layer import DecodeChain
    ys = [torch.empty((B, E), device=dev, dtype=torch.float32) for _ in range(NL)]
    chains = {}
    use_chain = world == 1 and NL > 1 and not args.no_chain and DecodeChain(layers).fused()

    def chain_of(start, cnt):
        if (start, cnt) not in chains:
            chains[(start, cnt)] = DecodeChain(layers[start:start + cnt])
        return chains[(start, cnt)]

    def run_steps(i0, n):
        """layer steps i0 .. i0 + n - 1 (step i on layer i mod NL)"""
        j = i0
        while j < i0 + n:
            start = j % NL
            if use_chain:
                cnt = min(NL - start, i0 + n - j)
                chain_of(start, cnt).step(xs[j // NL], ys[start:start + cnt])
            else:
                cnt = 1
                # eager launches (PDL-chained): a captured graph is bound to its
                # buffers, and layer 0's token changes every pass
                layers[start].step(xs[j // NL] if start == 0 else ys[start - 1], ys[start], graph=False)
                if comm is not None:
                    comm.allreduce_(ys[start])
            j += cnt

    # setup, untimed: each layer's first step sizes its workspaces and folds
    # its M_QK (host work with synchronising allocations)
    for li in range(NL):
        layers[li].step(xs[0], y)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    run_steps(0, W)
    # chains: the timed steps start on layer 0 (whole 8-layer chains; the
    # alignment steps are extra untimed warm-up) and every chain object they
    # use exists before the clock starts
    W0 = W + ((-W) % NL if use_chain else 0)
    run_steps(W, W0 - W)
    if use_chain:
        j = W0
        while j < W0 + K:
            cnt = min(NL - j % NL, W0 + K - j)
            chain_of(j % NL, cnt)
            j += cnt
    torch.cuda.synchronize()
    # soak: keep the GPU under the same load (the attention kernel, no append)
    # while the clock sampler collects samples around the timed region
    t_s = time.time()
    while time.time() - t_s < args.soak_ms / 1e3:
        for _ in range(50):
            layer.attention_only(out)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a ~0.2 ms device-side delay ahead of the start event: the host enqueues
    # the timed launches while it runs, so the device-timed value holds the K
    # steps' device time, not the first launch's host latency (e2e keeps it)
    if not args.no_predelay:
        torch.cuda._sleep(400_000)
    ev0.record(stream)
    run_steps(W0, K)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    clocks = sampler.stop()
    L_mid = pre + 1 + (W0 + K // 2) // NL + 1  # mean context of the timed steps (rows attended)
    ms_t = torch.tensor([ms_total], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total = float(ms_t.item())
    ms_step = ms_total / K
    value = B / (ms_step / 1e3)
    launches = 0
    j = W0
    while j < W0 + K:
        start = j % NL
        cnt = min(NL - start, W0 + K - j) if use_chain else 1
        launches += 1 if use_chain else layer.launches_per_step()
        j += cnt

    # ---- the same layer steps as one launch each (no chaining), for reference
    single = None
    if use_chain:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(NL):
            layers[i].step(xs[0], ys[i])
        torch.cuda.synchronize()
        if not args.no_predelay:
            torch.cuda._sleep(400_000)  # (as the timed chains: the launches enqueue behind it)
        s0.record(stream)
        for i in range(K):
            layers[i % NL].step(xs[i // NL] if i % NL == 0 else ys[i % NL - 1], ys[i % NL])
        s1.record(stream)
        torch.cuda.synchronize()
        single = s0.elapsed_time(s1) / K

    # ---- dominant kernel alone: decode attention (same stream, CUDA events)
    R = 20
    for _ in range(3):
        layer.attention_only(out)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(R):
        layer.attention_only(out)
    a1.record(stream)
    torch.cuda.synchronize()
    attn_ms = a0.elapsed_time(a1) / R
    attn_bytes, step_bytes = algorithmic_bytes(cfg, B, nh_g, L_mid)
    peak, peak_kind = measured_peak()
    achieved = attn_bytes / (attn_ms / 1e3) / 1e9
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    fused = layer.launches_per_step() == 1

    def traffic_of(fname):
        tp = os.path.join(ROOT, "profiles", fname)
        try:
            with open(tp) as fh:
                return json.load(fh).get(cfg_name)
        except Exception:
            return None

    # ---- end to end through the public API with host buffers
    xh = torch.empty((B, E), dtype=torch.float32).pin_memory()
    yh = torch.empty((B, E), dtype=torch.float32).pin_memory()
    xh.copy_(xs[0].cpu())
    xd = torch.empty((B, E), device=dev, dtype=torch.float32)
    yd = torch.empty((B, E), device=dev, dtype=torch.float32)
    Ke = max(3, min(K, 100))  # host-step wall time is noisy: time as many steps as the device run
    e2e_ms = None
    e2e_unit_layers = NL if use_chain else 1  # layer steps per host call
    if max(lay.length() for lay in layers) + Ke // NL + NL + 4 < cap:
        full = chain_of(0, NL) if use_chain else None

        def e2e_step(i):
            if use_chain:
                # one token through the NL chained layers: x in, the last y out
                full.step_host(xh.numpy(), yh.numpy())
                return
            lay = layers[i % NL]
            if comm is None:
                lay.step_host(xh.numpy(), yh.numpy())
            else:
                xd.copy_(xh, non_blocking=True)
                lay.step(xd, yd)
                comm.allreduce_(yd)
                yh.copy_(yd, non_blocking=True)
                stream.synchronize()
        ncalls = max(3, Ke // e2e_unit_layers)
        for i in range(NL if not use_chain else 1):  # first calls size workspaces / resolve the mapped pointers
            e2e_step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_e = time.perf_counter()
        for i in range(ncalls):
            e2e_step(i)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t_e) * 1e3 / (ncalls * e2e_unit_layers)
        et = torch.tensor([e2e_ms], device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_ms = float(et.item())

    # ---- the paper's comparison point: dense layer over the full KV cache with
    # Flash Decoding = torch SDPA, same shape and batch
    baselines = {}
    if world == 1 and not args.no_baselines:
        for name, fn in (("flash_decoding_sdpa", flash_decoding_baseline),
                         ("shared_latent_materialize", shared_latent_baseline)):
            try:
                b_ = fn(cfg, B, nh_g, L, dev)
                b_["speedup_of_ours"] = round(b_["us_per_layer"] / (ms_step * 1e3), 3)
            except Exception as e:  # reported, never the target
                b_ = {"unavailable": str(e)[:200]}
            baselines[name] = b_

    res = None
    if rank == 0:
        res = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": round(ms_step, 5),
            "us_per_layer": round(ms_step * 1e3, 2),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": {"bf16": "bf16 storage / fp32 accumulate", "f32": "f32",
                      "i8": "int8 (W8A8, int32 accumulate)", "i4": "int4 weights / int8 act"}[cfg["weights"]],
            "data": "synthetic (random-init factors, decode-bench recipe; random tokens)",
            "config": {"workload": cfg_name, "embed_dim": E, "heads": cfg["nh"], "heads_per_gpu": nh_g,
                       "head_dim": H, "rank": cfg["r"], "global_batch": B, "ctx": L_mid,
                       "ctx_range": [L + 0, layer.length()], "cache_dtype": cfg["cache"],
                       "weight_dtype": cfg["weights"], "parallelism": f"heads/{world}",
                       "step": "append(x.A_qkv) + fused decode attention + O-proj"
                               + (" + NCCL all-reduce" if world > 1 else ""),
                       "l2": l2_statement(NL, attn_bytes, step_bytes, l2_bytes),
                       "layers": NL,
                       "launch": (f"the {NL} rotating layers chained (layer l+1's token = layer l's y): one "
                                  f"persistent kernel per pass over them (wsvd_chain_step); {launches} launches "
                                  f"for the {K} timed layer steps, the first on layer 0 ({W0 - W} extra untimed "
                                  f"warm-up steps align it)" if use_chain else layer.step_kind()),
                       "timing": ("CUDA events around exactly the K steps, synchronised on both sides; "
                                  + ("a 0.2 ms device delay ahead of the start event lets the host enqueue the "
                                     "launches first (the value is device time; e2e includes host latency)"
                                     if not args.no_predelay else "the timed region starts on an idle device"))},
            "roofline": ({"bound": "hbm", "kernel": "layer_step_kernel (whole step: projection, append, "
                                                    "attention, merge, O-projection)",
                          "achieved": round(step_bytes / (ms_step / 1e3) / 1e9, 1), "peak": peak,
                          "peak_kind": peak_kind, "unit": "GB/s",
                          "frac": round(step_bytes / (ms_step / 1e3) / 1e9 / peak, 4),
                          "traffic": traffic_of("step_traffic.json"), "algorithmic_bytes": int(step_bytes),
                          "launch_us": round(ms_step * 1e3, 2),
                          "attention_kernel_alone": {"kernel": "decode_attn_kernel + attn_combine_kernel",
                                                     "us": round(attn_ms * 1e3, 2),
                                                     "algorithmic_bytes": int(attn_bytes),
                                                     "achieved": round(achieved, 1),
                                                     "frac": round(achieved / peak, 4),
                                                     "traffic": traffic_of("attn_traffic.json")}}
                         if fused else
                         {"bound": "hbm", "kernel": "decode_attn_kernel", "achieved": round(achieved, 1),
                          "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                          "frac": round(achieved / peak, 4), "traffic": traffic_of("attn_traffic.json"),
                          "attn_us": round(attn_ms * 1e3, 2), "algorithmic_bytes": int(attn_bytes),
                          "step_algorithmic_bytes": int(step_bytes),
                          "step_frac": round(step_bytes / (ms_step / 1e3) / 1e9 / peak, 4)}),
            "clocks": clocks,
            "baselines": baselines,
            "gpu_launches": launches,
            "single_layer_launches": ({"ms_per_step": round(single, 5), "tokens_per_s": round(B / (single / 1e3), 1),
                                       "note": "the same layer steps, one wsvd_layer_step launch each"}
                                      if single is not None else None),
            "e2e": {"value": round(B / (e2e_ms / 1e3), 1) if e2e_ms else None, "unit": "tokens/s",
                    "ms_per_step": round(e2e_ms, 4) if e2e_ms else None,
                    "h2d_bytes_per_step": B * E * 4 // e2e_unit_layers,
                    "d2h_bytes_per_step": B * E * 4 // e2e_unit_layers,
                    "api": (f"wsvd_chain_step_host (C ABI): one token of every sequence through the {NL} "
                            f"chained layers per call, pinned x in / last y out moved by the kernel's own bus "
                            f"loads/stores; per layer step = call time / {NL}, bytes per layer step = "
                            f"x + y bytes / {NL}") if use_chain else
                           (("wsvd_layer_step_host (C ABI; pinned x/y moved by the fused kernel's own "
                             "bus loads/stores)" if fused else "wsvd_layer_step_host (C ABI; copy engine)")
                            if world == 1 else "DecodeLayer.step + NCCL")},
        }
    if not args.no_strong:
        strong = strong_scaling_point(args, world, rank, local, comm)
        if res is not None:
            res["strong_scaling"] = strong
    del layer, layers
    return res


STRONG_CONFIG = "13b-r48-b64-ctx8k-w4a8-i8cache"


def strong_scaling_point(args, world, rank, local, comm, steps=20, warmup=5):
    """north_star config 4 with a FIXED global batch: the 40 heads of the 13B
    layer (r48, W4A8, INT8 cache, B = 64, ctx 8K) sharded over the N GPUs of
    this run, one NCCL all-reduce of the O-projection partials per step; per
    GPU 2.1 GB / N of cache (1057 / 529 / 265 MB at
    N = 2 / 4 / 8).  Timed like the headline (CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2604_02570_b200.layer import DecodeLayer
    from paper_2604_02570_b200.sharding import shard_factors, shard_oproj
    cfg = CONFIGS[STRONG_CONFIG]
    E, H, B, L = cfg["E"], cfg["H"], cfg["B"], cfg["L"]
    nh_g = cfg["nh"] // world
    dev = torch.device("cuda", local)
    t0 = time.time()
    f, w_o = synthetic_layer(cfg, seed=args.seed + 1)
    lay = DecodeLayer(shard_factors(f, world, rank), shard_oproj(w_o, cfg["nh"], H, world, rank), batch=B,
                      capacity=L + steps + warmup + 8, cache_dtype=cfg["cache"], weight_dtype=cfg["weights"],
                      oproj_dtype="bf16", device=local, head_offset=rank * nh_g)
    lay.fill_synthetic(L - 1 - warmup, seed=3)
    g = torch.Generator(device=dev)
    g.manual_seed(77 + args.seed)
    xs = torch.randn((warmup + steps, B, E), generator=g, device=dev)
    y = torch.empty((B, E), device=dev)
    stream = torch.cuda.current_stream()

    def step(i):
        lay.step(xs[i], y)
        if comm is not None:
            comm.allreduce_(y)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        step(warmup + i)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    _, step_bytes = algorithmic_bytes(cfg, B, nh_g, L)
    peak, peak_kind = measured_peak()
    out = {"workload": STRONG_CONFIG, "scaling": "strong", "global_batch": B, "heads_per_gpu": nh_g,
           "n_gpus": world, "ctx": L, "us_per_layer": round(ms * 1e3, 2),
           "tokens_per_s": round(B / (ms / 1e3), 1),
           "hbm_frac_per_gpu": round(step_bytes / (ms / 1e3) / 1e9 / peak, 4), "peak_kind": peak_kind,
           "algorithmic_bytes_per_gpu": int(step_bytes), "launches_per_step": lay.launches_per_step(),
           "step": "append + attention + O-proj" + (" + NCCL all-reduce" if world > 1 else ""),
           "setup_s": round(time.time() - t0, 1)}
    del lay
    torch.cuda.empty_cache()
    return out


def shared_latent_baseline(cfg, B, nh_g, L, dev, steps=5):
    """The paper's "W/o per-head" point: one shared latent (width nh*r, the same
    cache bytes) with the naive materialising schedule (baselines.py)."""
    import torch

    from paper_2604_02570_b200.baselines import SharedLatentLayer
    E, H, r = cfg["E"], cfg["H"], cfg["r"]
    base = SharedLatentLayer(E, nh_g, H, nh_g * r, B, L + steps + 8, device=dev.index)
    base.fill(L - 1)
    x = torch.randn((B, E), device=dev, dtype=torch.bfloat16)
    y = torch.empty((B, E), device=dev, dtype=torch.bfloat16)
    # every timed step re-runs position L-1 (identical work and tensor shapes,
    # so the allocator holds steady across the large materialised K / V)
    run = base.step_fn(x, y, L - 1)
    for i in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    out = {"us_per_layer": round(us, 2), "tokens_per_s": round(B / (us / 1e6), 1),
           "latent_cache_bytes": base.latent_bytes(L), "shared_rank": nh_g * r, "dtype": "bf16",
           "kernels": "cuBLAS GEMMs materialising every head's K / V from the shared latent + SDPA",
           "source": "PAPER.md:1302-1327 (W/o per-head); decode.cpp:330-390 shared_decode_step(materialize)"}
    del base
    torch.cuda.empty_cache()
    return out


def flash_decoding_baseline(cfg, B, nh_g, L, dev, steps=20):
    """Dense full-rank layer step with SDPA over the full KV cache (library
    kernels; paper_2604_02570_b200/baselines.py), CUDA-graph replayed, timed
    with CUDA events at the bench's context length."""
    import torch

    from paper_2604_02570_b200.baselines import DenseFlashDecodeLayer
    E, H = cfg["E"], cfg["H"]
    base = DenseFlashDecodeLayer(E, nh_g, H, B, L + steps + 8, device=dev.index)
    base.fill(L - 1)
    x = torch.randn((B, E), device=dev, dtype=torch.bfloat16)
    y = torch.empty((B, E), device=dev, dtype=torch.bfloat16)
    fns = [base.step_fn(x, y, L - 1 + i) for i in range(steps)]
    for fn in fns[:3]:
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        for fn in fns:
            fn()
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    out = {"us_per_layer": round(us, 2), "tokens_per_s": round(B / (us / 1e6), 1),
           "kv_cache_bytes": base.kv_bytes(L), "dtype": "bf16",
           "kernels": "cuBLAS QKV / O GEMMs + torch.nn.functional.scaled_dot_product_attention over the full KV cache",
           "source": "PAPER.md:685-690 (Flash Decoding = SDPA, full KV cache)"}
    del base, graph
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------- config 5 stack ---
def run_stack(args, cfg_name, cfg):
    """pipe::decode_factored (pipeline.cpp:304-339) over `layers` WSVD layers +
    the toy FFN, one token for every sequence per step, the whole stack step
    replayed as one CUDA graph.  Caches are filled with synthetic latents
    (wsvd_cache_fill_synthetic; a 32K-token prompt through the projection
    is not part of the decode step being measured)."""
    import torch
    import torch.distributed as dist

    from paper_2604_02570_b200 import _native as N
    from paper_2604_02570_b200.layer import DecodeLayer
    from paper_2604_02570_b200.sharding import NcclComm
    from paper_2604_02570_b200.stack import DecodeStack

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N.lib()
    E, H, B, L, nl = cfg["E"], cfg["H"], cfg["B"], cfg["L"], cfg["layers"]
    shard_of = cfg["shard_of"]
    nh_g = cfg["nh"] // shard_of
    sub = dict(cfg, nh=nh_g)
    W, K = args.warmup, args.steps
    cap = L + W + K + 8
    dev = torch.device("cuda", local)
    t0 = time.time()
    layers = []
    for li in range(nl):
        f, w_o = synthetic_layer(sub, seed=args.seed * 1000 + rank * 100 + li)
        lay = DecodeLayer(f, w_o, batch=B, capacity=cap, cache_dtype=cfg["cache"], weight_dtype=cfg["weights"],
                          oproj_dtype="bf16", device=local, head_offset=rank * nh_g)
        lay.fill_synthetic(L - 1 - W, seed=li + 1)
        layers.append(lay)
    comm = NcclComm(world, rank, local) if world > 1 else None
    stack = DecodeStack(layers, comm=comm, seed=args.seed)
    log(f"[rank {rank}] stack setup {time.time() - t0:.1f}s")
    x = torch.randn((B, E), device=dev)
    y = torch.empty((B, E), device=dev)
    for _ in range(W):  # warm-up (sizes every workspace) -- outside any graph
        stack.step(x, y)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        stack.step(x, y)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    ev0.record(stream)
    for _ in range(K):
        graph.replay()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms_t = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / K
    for lay in layers:
        lay.sync_length()
    L_end = layers[0].length()
    _, lbytes = algorithmic_bytes(sub, B, nh_g, L_end - K // 2)
    step_bytes = nl * lbytes + stack.ffn_bytes()
    peak, peak_kind = measured_peak()
    achieved = step_bytes / (ms_step / 1e3) / 1e9
    res = None
    if rank == 0:
        res = {
            "metric": METRIC, "value": round(B / (ms_step / 1e3), 1), "unit": "tokens/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": round(ms_step, 4),
            "us_per_layer": round(ms_step * 1e3 / nl, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 storage / fp32 accumulate",
            "data": "synthetic (random-init factors and FFN; synthetic N(0,1) latent caches)",
            "config": {"workload": cfg_name, "layers": nl, "embed_dim": E, "heads": cfg["nh"],
                       "heads_per_gpu": nh_g, "head_dim": H, "rank": cfg["r"], "global_batch": B,
                       "ctx": L_end - K // 2, "ffn": "toy tanh FFN 2E (pipeline.cpp:330-334): wsvd_ffn_forward, two tcgen05 GEMMs "
                              "(gemm_tc.cu), bf16 weights, replicated",
                       "parallelism": f"heads/{shard_of} (each GPU one {shard_of}-way head shard; {world} of "
                                      f"the {shard_of} shards run)",
                       "l2": f"inputs larger than L2 ({torch.cuda.get_device_properties(dev).L2_cache_size / 1e6:.0f} MB): "
                             f"{nl * lbytes / 1e9:.1f} GB of latent caches per GPU",
                       "launch": "whole 32-layer step captured as one CUDA graph"},
            "roofline": {"bound": "hbm", "kernel": "whole stack step (all kernels)", "achieved": round(achieved, 1),
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": None, "algorithmic_bytes": int(step_bytes)},
            "clocks": clocks,
            "gpu_launches": K * nl * layers[0].launches_per_step(),
            "e2e": {"value": None, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "note": "config-5 line: device-resident stack step only"},
        }
    del graph, stack, layers
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res


# ------------------------------------------------------- CPU baselines ----
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_rate(cfg, B, steps, warmup, threads, L=None):
    """The reference's own fused_decode_step + append_token (oracle/_ref, compiled
    from the reference sources) on the host cores; returns (tokens/s, kind, detail)."""
    from oracle import oracle as O
    L = L or cfg["L"]
    if O.ref_available():
        R = O.ref()
        h = R.ref_baseline_create(cfg["E"], cfg["H"], cfg["nh"], cfg["r"], B, L, 32, 0, threads)
        if not h:
            raise RuntimeError(R.ref_last_error().decode())
        for _ in range(warmup):
            R.ref_baseline_step(h, threads)
        ms = [R.ref_baseline_step(h, threads) for _ in range(steps)]
        R.ref_baseline_destroy(h)
        kind = "reference"
    else:
        # the oracle port (same algorithm, plain C), batched over (sequence, head)
        lay = O.bench_layer(cfg["E"], cfg["H"], cfg["nh"], cfg["r"])
        cap = L + warmup + steps + 2
        ck = np.random.default_rng(0).standard_normal((B, cfg["nh"], cap, cfg["r"]))
        cv = np.random.default_rng(1).standard_normal((B, cfg["nh"], cap, cfg["r"]))
        ms = []
        length = L - 1
        for i in range(warmup + steps):
            x = np.random.default_rng(2 + i).standard_normal((B, cfg["E"]))
            t = time.perf_counter()
            q = O.batched_append(lay, ck, cv, length, x, threads)
            O.batched_decode(lay, ck, cv, length + 1, q, 32, threads)
            length += 1
            if i >= warmup:
                ms.append((time.perf_counter() - t) * 1e3)
        kind = "port"
    med = statistics.median(ms)
    return B / (med / 1e3), kind, med


def run_reference_arm(args, cfg_name, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    threads = cpu_threads()
    B = cfg["B"] * world
    rate, kind, med = cpu_reference_rate(cfg, B, args.steps, args.warmup, threads)
    return {
        "metric": METRIC, "value": round(rate, 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(med, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (decode-bench recipe factors; N(0,1) latent prefill)",
        "impl": "reference",
        "config": {"workload": cfg_name, "embed_dim": cfg["E"], "heads": cfg["nh"],
                   "head_dim": cfg["H"], "rank": cfg["r"], "global_batch": B, "ctx": cfg["L"],
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": round(rate, 3), "unit": "tokens/s", "cores": threads, "kind": kind,
                         "sample": f"full workload: {B} sequences x {cfg['nh']} heads, ctx {cfg['L']}, "
                                   f"append_token + fused_decode_step per (sequence, head), fp64"},
        "e2e": {"value": round(rate, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS) + sorted(STACK_CONFIGS))
    ap.add_argument("--soak-ms", type=float, default=1500.0,
                    help="untimed attention load before the timed region while clocks are sampled")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-strong", action="store_true",
                    help="skip the config-4 strong-scaling point (fixed B = 64, heads over the N GPUs)")
    ap.add_argument("--layers", type=int, default=32,
                    help="rotating layers (own weights and cache each; 32 = LLaVA-7B's depth, one chain launch "
                         "per token through all of them): step i runs layer i mod n")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-predelay", action="store_true",
                    help="start the timed region on an idle device (the first launch's host latency inside it)")
    ap.add_argument("--no-chain", action="store_true",
                    help="one launch per layer step instead of the fused layer chain")
    ap.add_argument("--cpu-sample-seqs", type=int, default=2)
    ap.add_argument("--no-baselines", action="store_true", help="skip the Flash Decoding (SDPA) comparison")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        raise SystemExit("--warmup must be >= 3")
    if args.config in STACK_CONFIGS:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config-5 stack line: the reference arm is "
                              "measured on the single-layer headline workload"}), flush=True)
            return
        res = run_stack(args, args.config, STACK_CONFIGS[args.config])
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        res = run_reference_arm(args, args.config, cfg)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    res = run_ours(args, args.config, cfg)
    if dist_env()[0] > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if res is None:
        return
    if args.gpus == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        try:
            bs = args.cpu_sample_seqs
            rate, kind, med = cpu_reference_rate(cfg, bs, 2, 1, threads)
            res["cpu_baseline"] = {
                "value": round(rate, 3), "unit": "tokens/s", "cores": threads, "kind": kind,
                "sample": f"{bs} sequences x {cfg['nh']} heads at ctx {cfg['L']} (same per-sequence "
                          f"work as the workload; tokens/s = sequences / step time), median of 2 steps, fp64",
                "ms_per_step": round(med, 2)}
        except Exception as e:  # the baseline is reported, never the target
            res["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": threads,
                                   "kind": "unavailable", "sample": str(e)[:200]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
