"""A few fused layer steps at a bench configuration (synthetic latents), for
ncu captures and compute-sanitizer runs of the production kernel.

    python tools/one_step.py [--config 7b-r32-b16-ctx4k-bf16] [--steps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_02570_b200.layer import DecodeLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    f, w_o = bench.synthetic_layer(cfg)
    B, E, L = cfg["B"], cfg["E"], cfg["L"]
    layer = DecodeLayer(f, w_o, batch=B, capacity=L + args.steps + 8, cache_dtype=cfg["cache"],
                        weight_dtype=cfg["weights"], oproj_dtype="bf16")
    layer.fill_synthetic(L - 1, seed=1)
    x = torch.randn((B, E), device="cuda")
    y = torch.empty((B, E), device="cuda")
    for _ in range(args.steps):
        layer.step(x, y)
    torch.cuda.synchronize()
    print("steps", args.steps, "kind", layer.step_kind())


if __name__ == "__main__":
    main()
