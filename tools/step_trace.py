"""Phase timeline of the fused layer-step kernel (step.cu STEP_MARK points),
from %globaltimer stamps of every CTA: run with WSVD_STEP_TRACE=1.

    WSVD_STEP_TRACE=1 python tools/step_trace.py [--config ...]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("WSVD_STEP_TRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_02570_b200.layer import DecodeLayer  # noqa: E402

MARKS = ["entry", "griddep", "P1 done", "q count", "qt ready", "attn done", "merged", "G2 exit",
         "P3 staged", "end", "P3 item0 in", "attn start", "P3 item0 mma", "1st merge",
         "prep0 done", "w0 start", "w7 start", "stage0 in", "x staged", "ring items", "parked items", "ring item 0 out", "P0 valid", "G2 arrive", "P3 y sent/recv", "P3 own psum", "P3 done", "P3 w0-3 items", "P3 w4-7 items", "P3 bar (tid0)"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--per-sm", action="store_true")
    ap.add_argument("--save", default=None)
    ap.add_argument("--dump", action="store_true", help="every CTA's marks")
    ap.add_argument("--attn-only", action="store_true")
    ap.add_argument("--proj-only", action="store_true")
    ap.add_argument("--host", action="store_true", help="steps through wsvd_layer_step_host (pinned x / y)")
    ap.add_argument("--chain", type=int, default=0,
                    help="run N chained layers as one launch (wsvd_chain_step); the marks are those of the layer "
                         "WSVD_STEP_TRACE_LAYER (default the last); 'entry' = that layer's start")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    E, B, L = cfg["E"], cfg["B"], cfg["L"]
    f, w_o = bench.synthetic_layer(cfg)
    layer = DecodeLayer(f, w_o, batch=B, capacity=L + 64, cache_dtype=cfg["cache"], weight_dtype=cfg["weights"])
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for t0 in range(0, L - 1 - args.steps, 256):
        n = min(256, L - 1 - args.steps - t0)
        layer.prefill(torch.randn((n, B, E), generator=g, device=dev))
    x = torch.randn((B, E), generator=g, device=dev)
    y = torch.empty((B, E), device=dev)
    xh, yh = x.cpu().pin_memory(), torch.empty((B, E)).pin_memory()
    chain = None
    if args.chain > 1:
        from paper_2604_02570_b200.layer import DecodeChain
        more = []
        for li in range(1, args.chain):
            f2, w2 = bench.synthetic_layer(cfg, seed=li)
            lay2 = DecodeLayer(f2, w2, batch=B, capacity=L + 64, cache_dtype=cfg["cache"],
                               weight_dtype=cfg["weights"])
            lay2.fill_synthetic(L - 1 - args.steps, seed=li)
            more.append(lay2)
        chain = DecodeChain([layer] + more)
        ys = [torch.empty((B, E), device=dev) for _ in range(args.chain)]
    for _ in range(args.steps):
        if chain is not None:
            if args.host:
                chain.step_host(xh.numpy(), yh.numpy())
            else:
                chain.step(x, ys)
        elif args.host:
            layer.step_host(xh.numpy(), yh.numpy())
        else:
            layer.step(x, y, graph=False)
    torch.cuda.synchronize()
    raw = layer.debug_copy("trace").astype(np.int64)
    t = np.concatenate([raw[:, :10], raw[:, 12:12 + len(MARKS) - 10]], axis=1)
    smid, nu = raw[:, 10], raw[:, 11]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    if args.attn_only:  # attention CTAs only (nu > 0): the projection CTAs skip marks 3-5
        rel = rel[nu > 0]
    if args.proj_only:
        rel = rel[nu == 0]
    print(f"{'mark':10s} {'min':>8s} {'median':>8s} {'max':>8s}   (us from the first CTA's entry)")
    for k, name in enumerate(MARKS):
        col = rel[:, k]
        print(f"{name:10s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")
    if args.dump:
        print("cta smid " + " ".join(f"{n[:9]:>9s}" for n in MARKS))
        for i in range(rel.shape[0]):
            print(f"{i:3d} {smid[i]:4d} " + " ".join(f"{v:9.2f}" for v in rel[i]))
    if args.per_sm:
        # per-SM attention-phase duration (first segment's query -> attention
        # done) and segment count, by SM id; --save appends them for
        # cross-run comparisons (is a slow SM slow every step?)
        dur = rel[:, 5] - rel[:, 11]
        order = np.argsort(smid)
        print("smid segs attn_us")
        for i in order:
            print(f"{smid[i]:4d} {nu[i]:5d} {dur[i]:7.2f}")
        if args.save:
            with open(args.save, "a") as fh:
                fh.write(" ".join(f"{smid[i]}:{dur[i]:.3f}" for i in order) + "\n")


if __name__ == "__main__":
    main()
