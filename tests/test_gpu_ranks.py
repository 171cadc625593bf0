"""Per-head ranks up to the head width (a2): the reference accepts any rank
<= H (factorize.cpp:72-164; the paper's rho2 = 70 / 90 % points need r ~ 90 /
115 at H = 128).  Ragged ranks are zero-padded to one common
width (a multiple of 16, up to 128 on the device): bf16 and int8 caches take
every padded width up to 128, fp32 caches up to 64.

Each case prefills a cache through the device projection, appends one more
token, and checks against the oracle on the values the device stores:
the query (append_token, decode.cpp:127-153), the attention over the device's
latent rows (fused_decode_step, decode.cpp:155-206), and the layer step's y
(pipeline.cpp:320-329 with the folded W'_o)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import REL_TOL, oracle_step_y, rel_err_rows, to_factors

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _ragged(nh, rmax, seed):
    rng = np.random.default_rng(seed)
    ranks = [[int(rng.integers(rmax // 2, rmax + 1)) for _ in range(3)] for _ in range(nh)]
    ranks[0] = [rmax, rmax, rmax]  # the padded width is reached
    return ranks


@pytest.mark.parametrize("cache,weights,rmax", [
    ("bf16", "bf16", 64), ("bf16", "bf16", 96), ("bf16", "bf16", 128), ("bf16", "bf16", 80),
    ("f32", "f32", 48), ("f32", "f32", 64),
])
def test_large_ranks_float(cache, weights, rmax):
    from paper_2604_02570_b200.layer import DecodeLayer
    E, nh, H, B, L = 512, 8, 128, 3, 300
    rng = O.Rng(5000 + rmax + (cache == "f32"))
    lay = O.random_layer(rng, E, H, _ragged(nh, rmax, rmax))
    wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / math.sqrt(E)))
    rnd = O.bf16_round if weights == "bf16" else O.f32_round
    lb = lay.map(rnd)
    toks = rnd(rng.normal_matrix(L * B, E)).reshape(L, B, E).astype(np.float32)
    dev = torch.device("cuda", 0)
    mk = lambda: DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 8, cache_dtype=cache,  # noqa: E731
                             weight_dtype=weights, oproj_dtype="bf16")
    a, s = mk(), mk()
    R = a.rpad
    assert R == (rmax + 15) // 16 * 16
    pre = torch.from_numpy(toks[:-1]).to(dev)
    a.prefill(pre)
    s.prefill(pre)
    q = torch.empty((B, nh, H), device=dev)
    a.append(torch.from_numpy(toks[-1]).to(dev), q)
    out = torch.empty((B, nh, H), device=dev)
    a.attend(q, out)
    y = torch.empty((B, E), device=dev)
    s.step(torch.from_numpy(toks[-1]).to(dev), y)
    torch.cuda.synchronize()
    q, out, y = (t.cpu().numpy().astype(np.float64) for t in (q, out, y))
    for b in range(B):
        ck = np.stack([a.read_latents(b, h)[0][:, :lay.rmax] for h in range(nh)])
        cv = np.stack([a.read_latents(b, h)[1][:, :lay.rmax] for h in range(nh)])
        for h in range(nh):  # zero padding stays zero
            assert not a.read_latents(b, h)[0][:, lay.ranks[h, 1]:].any()
        nk, nv = np.zeros((nh, 1, lay.rmax)), np.zeros((nh, 1, lay.rmax))
        q_ref = O.append_token(lb, nk, nv, 0, toks[-1, b].astype(np.float64))
        assert rel_err_rows(q[b], q_ref) <= REL_TOL, f"query b={b}"
        ref = O.fused_decode_step(lb, ck, cv, L, q[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL, f"attention b={b}"
        sk = np.stack([s.read_latents(b, h)[0][:, :lay.rmax] for h in range(nh)])
        sv = np.stack([s.read_latents(b, h)[1][:, :lay.rmax] for h in range(nh)])
        y_ref = oracle_step_y(lb, sk, sv, L, q_ref, wo, R)
        assert rel_err_rows(y[b:b + 1], y_ref[None]) <= REL_TOL, f"y b={b}"


@pytest.mark.parametrize("weights,rmax", [("i8", 96), ("i4", 128), ("i8", 64)])
def test_large_ranks_int8_cache(weights, rmax):
    from paper_2604_02570_b200.layer import DecodeLayer
    from tests.test_gpu_int import quant_layer
    E, nh, H, B, L = 512, 4, 128, 2, 200
    rng = O.Rng(6000 + rmax)
    lay = O.random_layer(rng, E, H, _ragged(nh, rmax, rmax + 1))
    quant, deq_b = quant_layer(lay, 8 if weights == "i8" else 4)
    deq = O.Layer(lay.A, deq_b, lay.ranks)
    wo = O.bf16_round(rng.normal_matrix(nh * H, E, 1.0 / math.sqrt(E)))
    toks = rng.normal_matrix(L * B, E).reshape(L, B, E).astype(np.float32)
    dev = torch.device("cuda", 0)
    layer = DecodeLayer(to_factors(lay), wo, batch=B, capacity=L + 8, cache_dtype="i8", weight_dtype=weights,
                        oproj_dtype="bf16", quantized=quant)
    R = layer.rpad
    layer.prefill(torch.from_numpy(toks[:-1]).to(dev))
    q = torch.empty((B, nh, H), device=dev)
    layer.append(torch.from_numpy(toks[-1]).to(dev), q)
    out = torch.empty((B, nh, H), device=dev)
    layer.attend(q, out)
    torch.cuda.synchronize()
    q, out = q.cpu().numpy().astype(np.float64), out.cpu().numpy().astype(np.float64)
    for b in range(B):
        ck = np.stack([layer.read_latents(b, h)[0][:, :lay.rmax] for h in range(nh)])
        cv = np.stack([layer.read_latents(b, h)[1][:, :lay.rmax] for h in range(nh)])
        ref = O.fused_decode_step(deq, ck, cv, L, q[b], 32)
        assert rel_err_rows(out[b], ref) <= REL_TOL, f"attention b={b}"
    assert R == (rmax + 15) // 16 * 16
