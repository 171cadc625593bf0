"""Small invocations of the kernels changed this round, for compute-sanitizer:
the fused step at a two-chunk shape (CTA-pair clusters, parked P1 items, full
first-stage copies), the int8-cache attention (1024-token stages, helper-warp
merge) and the fp32 row GEMV.

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2604_02570_b200.layer import DecodeLayer  # noqa: E402
from tests.helpers import to_factors  # noqa: E402
from tests.test_gpu_int import quant_layer  # noqa: E402

dev = torch.device("cuda", 0)
rng = O.Rng(5)

# fused step, 512 (sequence, head) pairs -> two chunks -> CTA pairs
E, nh, H, r, B, L = 1024, 32, 128, 32, 16, 300
lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(E)))
layer = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 4, cache_dtype="bf16", weight_dtype="bf16")
layer.fill_synthetic(L - 2)
x = torch.randn((B, E), device=dev)
y = torch.empty((B, E), device=dev)
for _ in range(2):
    layer.step(x, y)
torch.cuda.synchronize()
print("fused step ok", float(y.abs().max()))

# int8 cache + W8A8, 148 pairs (single chunk: in-kernel merge), ragged last stage
E, nh, B, L = 512, 4, 37, 1500
lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
quant, _ = quant_layer(lay, 8)
wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(nh * H)))
il = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 4, cache_dtype="i8", weight_dtype="i8", quantized=quant)
il.fill_synthetic(L - 1)
x = torch.randn((B, E), device=dev)
y = torch.empty((B, E), device=dev)
il.step(x, y, graph=False)
torch.cuda.synchronize()
print("int8 step ok", float(y.abs().max()))

# fp32 weights, one sequence: the row GEMV and the 4-CTA-cluster attention
# (chunks merged through DSMEM), at a length with empty trailing chunks too
E, nh, B = 512, 32, 1
lay = O.random_layer(rng, E, H, [[r, r, r]] * nh)
wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / np.sqrt(nh * H)))
for L in (200, 40):
    fl = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 4, cache_dtype="f32", weight_dtype="f32")
    fl.fill_synthetic(L - 1)
    y = torch.empty((B, E), device=dev)
    fl.step(torch.randn((B, E), device=dev), y, graph=False)
    torch.cuda.synchronize()
    print("fp32 step ok", L, float(y.abs().max()))
