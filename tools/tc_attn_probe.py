"""The explicit tcgen05 key-reconstruction attention (attn_tc.cu) at the
headline workload: device time over reps (CUDA events) -- the target of
`ncu -k regex:decode_attn_tc`.  python tools/tc_attn_probe.py [--reps 20]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_02570_b200.layer import DecodeLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = bench.CONFIGS[bench.DEFAULT_CONFIG]
    f, w = bench.synthetic_layer(cfg)
    B, E, L, nh, H = cfg["B"], cfg["E"], cfg["L"], cfg["nh"], cfg["H"]
    lay = DecodeLayer(f, w, batch=B, capacity=L + 8, cache_dtype="bf16", weight_dtype="bf16", attention="explicit_tc")
    lay.fill_synthetic(L - 1, seed=1)
    dev = torch.device("cuda", 0)
    q = torch.randn((B, nh, H), device=dev)
    out = torch.empty((B, nh, H), device=dev)
    for _ in range(3):
        lay.attend(q, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        lay.attend(q, out)
    e1.record()
    torch.cuda.synchronize()
    print(f"explicit tcgen05 attention (+ combine): {e0.elapsed_time(e1) * 1e3 / args.reps:.2f} us")
    lay.set_attention("absorbed")
    lay.attend(q, out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.reps):
        lay.attend(q, out)
    e1.record()
    torch.cuda.synchronize()
    print(f"absorbed attention (+ combine): {e0.elapsed_time(e1) * 1e3 / args.reps:.2f} us")


if __name__ == "__main__":
    main()
