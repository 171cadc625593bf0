"""Small invocations of this round's kernels for compute-sanitizer (memcheck,
racecheck of shared memory is not applicable to TMA / tcgen05 traffic):

    compute-sanitizer --tool memcheck python tools/sanitize_probe_r02.py

the layer chain (step.cu, 3 layers, CTA pairs, parked items across layers,
DSMEM O-projection reduction), the two-group chain (step2.cu, WSVD_CHAIN_PIPE
is read once: run a second process with it set), the tcgen05 GEMM through the
FFN (one and two K splits, 1 .. 200 rows), the tcgen05 prefill projection and
the TMA-ring fp32 GEMV."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2604_02570_b200.layer import DecodeChain, DecodeLayer  # noqa: E402
from paper_2604_02570_b200.stack import FeedForward, toy_ffn_weights  # noqa: E402
from tests.helpers import to_factors  # noqa: E402

dev = torch.device("cuda", 0)
rng = O.Rng(5)
# ---- chain: E 1024, 32 heads, B 16, three layers of different lengths
E, nh, B = 1024, 32, 16
layers = []
for L in (200, 70, 1):
    lay = O.random_layer(rng, E, 128, [[32, 32, 32]] * nh)
    wo = O.bf16_round(rng.normal_matrix(nh * 128, E, 1 / np.sqrt(E)))
    d = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 8, cache_dtype="bf16", weight_dtype="bf16")
    d.fill_synthetic(L, seed=L)
    layers.append(d)
ch = DecodeChain(layers)
x = torch.randn((B, E), device=dev)
ys = [torch.empty((B, E), device=dev) for _ in range(3)]
ch.step(x, ys)
ch.step(ys[-1], ys)
torch.cuda.synchronize()
# ---- FFN on tcgen05: 1 and 200 rows (two 128-row chunks; GEMM2 over K splits)
for M in (1, 200):
    ffn = FeedForward(*toy_ffn_weights(512, 1024, M))
    o = torch.randn((M, 512), device=dev)
    out = torch.empty_like(o)
    ffn.forward(o, out)
torch.cuda.synchronize()
# ---- tcgen05 prefill projection (>= 64 token rows) and the fp32 TMA GEMV (1 row)
lay = O.random_layer(rng, 1024, 128, [[32, 32, 32]] * 8)
p = DecodeLayer(to_factors(lay), None, batch=8, capacity=40, cache_dtype="bf16", weight_dtype="bf16")
p.prefill(torch.randn((16, 8, 1024), device=dev))
f = DecodeLayer(to_factors(lay), None, batch=1, capacity=8, cache_dtype="f32", weight_dtype="f32")
f.append(torch.randn((1, 1024), device=dev))
torch.cuda.synchronize()
print("probe ok")
