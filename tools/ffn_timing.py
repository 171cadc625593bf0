"""Device time of the toy FFN (wsvd_ffn_forward: two skinny GEMMs + split
reductions) at the config-5 shape: python tools/ffn_timing.py [--rows 128]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_02570_b200.stack import FeedForward, toy_ffn_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=128)
    ap.add_argument("--E", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    E, F, M = args.E, 2 * args.E, args.rows
    w1, w2 = toy_ffn_weights(E, F, 0)
    ffn = FeedForward(w1, w2)
    o = torch.randn((M, E), device="cuda")
    out = torch.empty_like(o)
    for _ in range(3):
        ffn.forward(o, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        ffn.forward(o, out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.reps
    print(f"FFN rows {M} E {E}: {us:.1f} us ({4 * E * F / us / 1e3:.0f} GB/s of bf16 weights)")
    a = o.to(torch.bfloat16)
    b1, b2 = torch.randn((E, F), device="cuda", dtype=torch.bfloat16), torch.randn((F, E), device="cuda", dtype=torch.bfloat16)
    e0.record()
    for _ in range(args.reps):
        torch.matmul(torch.tanh(a @ b1), b2)
    e1.record()
    torch.cuda.synchronize()
    print(f"cuBLAS (torch bf16): {e0.elapsed_time(e1) * 1e3 / args.reps:.1f} us")


if __name__ == "__main__":
    main()
