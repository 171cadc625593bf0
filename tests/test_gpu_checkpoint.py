"""Device layers loaded straight from a reference checkpoint
(wsvd_layer_load_checkpoint, csrc/checkpoint.cpp) behave exactly like layers
built from the same tensors through the regular upload path: fp64 factors
(bf16 storage) and the QAT export (int8 factors, Hadamard-rotated
activations, int8 cache), with the checkpoint's W_o rows, for a full head
range and a head shard."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "ckpt_e64")


@pytest.mark.parametrize("wd,cd,heads", [("bf16", "bf16", None), ("f32", "f32", (1, 3)), ("i8", "i8", None),
                                         ("i8", "i8", (2, 4))])
def test_checkpoint_layer_equals_uploaded_layer(wd, cd, heads):
    from paper_2604_02570_b200.checkpoint import Checkpoint
    from paper_2604_02570_b200.layer import DecodeLayer
    ck = Checkpoint(FIX)
    h0, h1 = heads or (0, ck.n_heads)
    B, L = 3, 40
    a = ck.decode_layer(1, batch=B, capacity=L + 4, cache_dtype=cd, weight_dtype=wd, heads=heads)
    quant = None
    if wd == "i8":
        quant = [[ck.head_quantized(1, h, role) for role in range(3)] for h in range(h0, h1)]
    w_o = ck.weight("layer1.w_o")[h0 * ck.head_dim:h1 * ck.head_dim]
    b = DecodeLayer(ck.factors(1, (h0, h1), quantized=wd == "i8"), w_o, batch=B, capacity=L + 4, cache_dtype=cd,
                    weight_dtype=wd, quantized=quant, head_offset=h0)
    dev = torch.device("cuda", 0)
    rng = O.Rng(31)
    toks = torch.from_numpy(rng.normal_matrix(L * B, ck.embed_dim).reshape(L, B, -1).astype(np.float32)).to(dev)
    a.prefill(toks[:-1])
    b.prefill(toks[:-1])
    ya = torch.empty((B, ck.embed_dim), device=dev)
    yb = torch.empty((B, ck.embed_dim), device=dev)
    a.step(toks[-1], ya)
    b.step(toks[-1], yb)
    torch.cuda.synchronize()
    assert torch.isfinite(ya).all()
    assert torch.equal(ya, yb)
    for hh in range(h1 - h0):
        assert np.array_equal(a.read_latents(1, hh)[0], b.read_latents(1, hh)[0])
