"""Device time of the fused layer chain (wsvd_chain_step) for chains of 1, 2,
4 and 8 layers at a bench workload: CUDA events over K launches each; the
marginal cost per added layer separates the per-layer time from the launch.

    python tools/chain_timing.py [--config ...] [--reps K]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_02570_b200.layer import DecodeChain, DecodeLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--only", type=int, default=0, help="time only the chain of this many layers")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    E, B, L = cfg["E"], cfg["B"], cfg["L"]
    n = args.layers
    cap = L + 8 * args.reps + 64
    layers = []
    for li in range(n):
        f, w = bench.synthetic_layer(cfg, seed=li)
        lay = DecodeLayer(f, w, batch=B, capacity=cap, cache_dtype=cfg["cache"], weight_dtype=cfg["weights"])
        lay.fill_synthetic(L - 1, seed=li + 1)
        layers.append(lay)
    dev = torch.device("cuda", 0)
    x = torch.randn((B, E), device=dev)
    ys = [torch.empty((B, E), device=dev) for _ in range(n)]
    for li in range(n):
        layers[li].step(x, ys[li], graph=False)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    for m in ([args.only] if args.only else [1, 2, 4, 8]):
        if m > n:
            break
        ch = DecodeChain(layers[:m])
        ch.step(x, ys[:m])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.reps):
            ch.step(x, ys[:m])
        e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / args.reps
        print(f"chain {m}: {us:8.2f} us per launch, {us / m:7.2f} us per layer", flush=True)
    if args.only:
        return
    # one launch per layer, same layers
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.reps):
        for li in range(n):
            layers[li].step(x if li == 0 else ys[li - 1], ys[li], graph=False)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"layer steps: {e0.elapsed_time(e1) * 1e3 / (args.reps * n):7.2f} us per layer")


if __name__ == "__main__":
    main()
