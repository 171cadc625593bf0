"""Per-operator device timing of the layer step.

Each operator is captured N times into a torch CUDA graph and replayed once
(CUDA events around the replay), so host launch overhead is excluded.

    python tools/timing.py [--config 7b-r32-b16-ctx4k-bf16] [--reps 20]
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--synthetic", action="store_true",
                    help="fill the cache with synthetic rows instead of a prefill (no prefill launches)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    E, H, B, L = cfg["E"], cfg["H"], cfg["B"], cfg["L"]
    f, w_o = bench.synthetic_layer(cfg)
    cap = L + 12 * args.reps + 64
    layer = DecodeLayer(f, w_o, batch=B, capacity=cap, cache_dtype=cfg["cache"],
                        weight_dtype=cfg["weights"])
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    if args.synthetic:
        layer.fill_synthetic(L - 1)
    else:
        for t0 in range(0, L - 1, 256):
            n = min(256, L - 1 - t0)
            layer.prefill(torch.randn((n, B, E), generator=g, device=dev))
    x = torch.randn((B, E), generator=g, device=dev)
    y = torch.empty((B, E), device=dev)
    q = torch.empty((B, cfg["nh"], H), device=dev)
    out = torch.empty((B, cfg["nh"], H), device=dev)
    torch.cuda.synchronize()

    ops = {
        "append_token (proj+epi)": lambda s: layer.append(x, None, stream=s),
        "attention (attn+combine)": lambda s: layer.attention_only(out, stream=s),
        "fused_decode_step": lambda s: layer.attend(q, out, stream=s),
        "layer_step": lambda s: layer.step(x, y, graph=False, stream=s),
    }
    side = torch.cuda.Stream()
    for name, fn in ops.items():
        fn(torch.cuda.current_stream())  # warm: workspaces, kernel attributes
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            for _ in range(args.reps):
                fn(side)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:28s} {e0.elapsed_time(e1) * 1e3 / args.reps:9.2f} us")


if __name__ == "__main__":
    main()
