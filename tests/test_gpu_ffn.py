"""GPU parity of the feed-forward (wsvd_ffn_forward, the toy model's
tanh(o . ff1) . ff2 of pipeline.cpp:330-334): the tcgen05 GEMMs (gemm_tc.cu,
TMA + TMEM) and, where E or F is not a multiple of 64, the mma.sync skinny
GEMM -- against numpy on the values the device stores (bf16 weights, bf16
o and hidden activations), within the north_star 1e-3, for 1 .. 300 rows
(more than one 128-row tile)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import REL_TOL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("E,F,M", [(512, 1024, 1), (512, 1024, 7), (512, 1024, 128), (256, 512, 300),
                                   (4096, 8192, 128), (320, 640, 16)])
def test_ffn_matches_numpy(E, F, M):
    from paper_2604_02570_b200.stack import FeedForward, toy_ffn_weights
    ff1, ff2 = toy_ffn_weights(E, F, E + M)
    ffn = FeedForward(ff1, ff2)
    rng = np.random.default_rng(M)
    o = rng.standard_normal((M, E)).astype(np.float32)
    out = torch.empty((M, E), device="cuda")
    ffn.forward(torch.from_numpy(o).cuda(), out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    h = np.tanh(O.bf16_round(o.astype(np.float64)) @ ff1.astype(np.float64))
    ref = O.bf16_round(h) @ ff2.astype(np.float64)
    err = np.abs(got - ref).max(axis=1) / np.abs(ref).max(axis=1)
    assert err.max() <= REL_TOL, f"{err.max():.2e}"


def test_ffn_output_may_alias_input():
    from paper_2604_02570_b200.stack import FeedForward, toy_ffn_weights
    E, F, M = 512, 1024, 200
    ffn = FeedForward(*toy_ffn_weights(E, F, 3))
    x = torch.randn((M, E), device="cuda")
    ref = torch.empty_like(x)
    ffn.forward(x, ref)
    ffn.forward(x, x)
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
